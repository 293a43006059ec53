"""FWI gradient validated as the gradient of the data misfit (Taylor test).

The reference has no FWI gradient; the paper names a
"gradient test" without defining it. The standard one, in
the style of adjoint_test_with (acoustic.cpp:239-270):

    J(m) = 1/2 || d(m) - d_obs ||^2     (forward receiver traces, eta fixed)
    g    = the gradient the FWI path returns for residual d(m) - d_obs
    e1(h) = | J(m + h dm) - J(m) |                 = O(h)
    e2(h) = | J(m + h dm) - J(m) - h <dJ/dm, dm> | = O(h^2)

With this code's definitions -- grad += u(t) * vtt(t), vtt the adjoint
wavefield's second difference times cm (oracle/sf_port.h) -- the gradient of
J is dJ/dm = -grad: the adjoint run injects +residual, so grad carries the
opposite sign. The tests check that sign and scale (a centred difference of J
agrees with -<grad, dm> to 1 %) and the second-order decay of e2 over
h = 1 .. 1/8 (below that the fp32 traces put a floor under J).

The CPU test pins the oracle's gradient (which the GPU path matches bitwise,
test_gpu_parity.py / test_gpu_configs.py); the GPU test runs the product's
FwiPlan at the C5 layout (301^3, order 8, 201 x 201 surface receivers).
"""
import numpy as np
import pytest


def _blob(shape, scale, center=None):
    """exp(-|x - center|^2 / scale), centre of the grid by default (separable)."""
    c = np.array(shape, np.float64) / 2.0 if center is None else np.asarray(center, np.float64)
    g = [np.exp(-(np.arange(n, dtype=np.float64) - c[a]) ** 2 / scale) for a, n in enumerate(shape)]
    return g[0][:, None, None] * g[1][None, :, None] * g[2][None, None, :]


def _taylor(J, J0, gdm, dm_scale=1.0):
    """e1, e2 over h = 1, 1/2, 1/4, 1/8 and the centred-difference ratio."""
    hs = [2.0 ** -k for k in range(4)]
    e1, e2 = [], []
    for h in hs:
        Jp = J(h)
        e1.append(abs(Jp - J0))
        e2.append(abs(Jp - J0 - h * gdm))
    fd = (J(0.25) - J(-0.25)) / 0.5
    return hs, e1, e2, fd


def _check(hs, e1, e2, fd, gdm):
    print(f"taylor: h={hs} e1={e1} e2={e2} centred_fd={fd} <dJ/dm,dm>={gdm}")
    assert abs(fd / gdm - 1.0) < 0.01, (fd, gdm)
    slopes2 = [np.log2(e2[i] / e2[i + 1]) for i in range(len(hs) - 1)]
    slopes1 = [np.log2(e1[i] / e1[i + 1]) for i in range(len(hs) - 1)]
    assert min(slopes2) > 1.8, slopes2        # second order
    assert 0.4 < slopes1[-1] < 1.3, slopes1   # first order (tends to 1)
    assert all(e2[i] < e1[i] for i in range(len(hs)))


def test_port_gradient_taylor(port):
    shape, order, nt, h, bw = (40, 44, 48), 8, 150, 10.0, 6
    lo, hi = port.smooth_extrema(shape, 0, shape[0], 11, sigma=4.0)
    m, eta = port.smooth_medium(shape, 0, shape[0], 11, lo, hi, sigma=4.0, boundary_width=bw)
    dt = min(0.4 * h / 4500.0, port.stable_dt(3, order, h, 4500.0, 4500.0))
    src_c = np.array([[12 * h, 22.3 * h, 24.1 * h]])
    rec_c = np.array([[10 * h, (8 + 2 * i + 0.3) * h, (9 + 2 * j + 0.6) * h]
                      for i in range(14) for j in range(14)])
    sci, sw = port.interp(src_c, h, shape)
    rci, rw = port.interp(rec_c, h, shape)
    src = np.array([port.ricker(15.0, t * dt, 1 / 15.0) for t in range(nt)], np.float32)[:, None]
    cf = port.coefs(3, order, True, dt, h)
    ca = port.coefs(3, order, False, dt, h)

    def fwd(mm):
        hist = np.zeros((nt + 2,) + shape, np.float32)
        rec = np.zeros((nt, len(rci)), np.float32)
        port.forward_history(cf, hist, mm, eta, src, sci, sw, rec, rci, rw, nt)
        return hist, rec
    _, dobs = fwd((m * (1 + 0.05 * _blob(shape, 40.0))).astype(np.float32))
    hist, d0 = fwd(m)
    res = (d0 - dobs).astype(np.float32)
    J0 = 0.5 * float(((d0.astype(np.float64) - dobs) ** 2).sum())
    v = np.zeros((3,) + shape, np.float32)
    g = np.zeros(shape, np.float32)
    s2 = np.zeros((nt, 1), np.float32)
    port.adjoint_gradient(ca, v, m, eta, hist, res, rci, rw, s2, sci, sw, g, nt)
    rng = np.random.default_rng(3)
    dm = (rng.standard_normal(shape) * m * 0.01).astype(np.float32)
    inner = tuple(slice(bw, -bw) for _ in shape)
    mask = np.zeros(shape, bool)
    mask[inner] = True
    dm[~mask] = 0
    gdm = -float((g.astype(np.float64) * dm).sum())  # dJ/dm = -grad

    def J(hh):
        _, d = fwd((m + hh * dm).astype(np.float32))
        return 0.5 * float(((d.astype(np.float64) - dobs) ** 2).sum())
    _check(*_taylor(J, J0, gdm), gdm)


@pytest.mark.gpu
def test_gpu_gradient_taylor_c5_layout():
    import bench
    import paper_1609_03361_b200 as sf
    shape, order, nt = (301, 301, 301), 8, 500
    bw, h = bench.BW, bench.H
    dt = min(0.4 * h / 4500.0, sf.api._stable_dt(3, order, h, 4500.0, 4500.0))
    sm = sf.SmoothMedium(shape=shape, boundary_width=bw, spacing=h,
                         **{k: v for k, v in bench.SMOOTH.items()})
    lo, hi = sm.extrema()
    m, eta = sm.generate(lo, hi)
    mid = shape[1] // 2
    src_c = [[(bw + 2) * h, mid * h, mid * h]]
    rec_c = [[(bw + 10) * h, (bw + i) * h, (bw + j) * h] for i in range(201) for j in range(201)]

    def interp(coords):
        cis, ws = zip(*[sf.interpolation_weights(cc, h, shape) for cc in coords])
        return np.array(cis, np.int32), np.array(ws, np.float32)
    sci, sw = interp(src_c)
    rci, rw = interp(rec_c)
    src = np.array([sf.ricker_wavelet(10.0, t * dt, 0.1) for t in range(nt)], np.float32)[:, None]
    plan = sf.FwiPlan(shape, order, nt, dt, h, 1, len(rec_c))
    zero = np.zeros((nt, len(rec_c)), np.float32)

    def traces(mm):
        rec, _, _, _ = plan.gradient(mm, eta, src, sci, sw, rci, rw, zero)
        return rec
    # the model error and the perturbation sit where the first arrivals and
    # their reflections reach the receivers within nt: a few tens of cells
    # below the source (a perturbation the data cannot see in nt steps would
    # leave J flat to first order and the test vacuous)
    dobs = traces((m * (1 + 0.05 * _blob(shape, 200.0, (bw + 24, mid + 8, mid - 6))))
                  .astype(np.float32)).astype(np.float64)
    d0 = traces(m)
    J0 = 0.5 * float(((d0 - dobs) ** 2).sum())
    assert J0 > 0
    res = (d0 - dobs).astype(np.float32)
    rec_out, grad, _, _ = plan.gradient(m, eta, src, sci, sw, rci, rw, res)
    assert np.array_equal(rec_out, d0)
    dm = (m * 0.01 * _blob(shape, 120.0, (bw + 20, mid, mid))).astype(np.float32)
    gdm = -float((grad.astype(np.float64) * dm).sum())
    assert abs(gdm) > 1e-3 * J0

    def J(hh):
        d = traces((m + hh * dm).astype(np.float32)).astype(np.float64)
        return 0.5 * float(((d - dobs) ** 2).sum())
    _check(*_taylor(J, J0, gdm), gdm)

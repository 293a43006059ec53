"""Seeded smooth random media (configs C3/C4/C5; csrc/medium.cu).

CPU tests pin the oracle's restatement (oracle/sf_port.c sfp_smooth_*) to the
properties the decomposition relies on: any depth slab generates exactly the
planes the single domain has, and slab extrema combine to the global ones.
GPU tests check the product generator against the restatement bitwise, for
host output, a plan's HBM fields, and depth slabs of a slab plan. The sponge
is build_medium's (acoustic.cpp:67-105) evaluated from global indices.
"""
import numpy as np
import pytest


def bits(a):
    return np.ascontiguousarray(a).view(np.uint32)


SHAPES = [(50, 40, 36), (23, 31, 17), (70, 12, 40)]


@pytest.mark.parametrize("shape", SHAPES)
def test_port_slabs_match_single_domain(port, shape):
    lo, hi = port.smooth_extrema(shape, 0, shape[0], 77)
    m, eta = port.smooth_medium(shape, 0, shape[0], 77, lo, hi, boundary_width=6)
    cuts = [0, shape[0] // 3, shape[0] // 3 + 5, shape[0]]
    los, his = [], []
    for b, e in zip(cuts[:-1], cuts[1:]):
        l2, h2 = port.smooth_extrema(shape, b, e, 77)
        los.append(l2)
        his.append(h2)
        ms, es = port.smooth_medium(shape, b, e, 77, lo, hi, boundary_width=6)
        assert np.array_equal(bits(ms), bits(m[b:e]))
        assert np.array_equal(bits(es), bits(eta[b:e]))
    assert min(los) == lo and max(his) == hi


def test_port_medium_range_and_sponge(port):
    shape = (60, 50, 44)
    lo, hi = port.smooth_extrema(shape, 0, shape[0], 5)
    m, eta = port.smooth_medium(shape, 0, shape[0], 5, lo, hi, boundary_width=8)
    v = 1.0 / np.sqrt(m.astype(np.float64))
    assert abs(v.min() - 1500.0) < 1e-2 and abs(v.max() - 4500.0) < 1e-1
    # eta = m * sigma(d): zero in the interior, positive in the sponge
    assert (eta[8:-8, 8:-8, 8:-8] == 0).all()
    assert (eta[0] > 0).all() and (eta[:, :, -1] > 0).all()
    # smooth: neighbouring cells differ by far less than the range
    assert np.abs(np.diff(v, axis=2)).max() < 0.1 * 3000.0
    # different seeds give different media
    lo2, hi2 = port.smooth_extrema(shape, 0, shape[0], 6)
    assert (lo2, hi2) != (lo, hi)


def test_port_taps_normalised(port):
    import ctypes as C
    g = np.zeros(129)
    rad = port.lib.sfp_smooth_taps(C.c_double(8.0), g)
    assert rad == 32
    assert abs(g[: 2 * rad + 1].sum() - 1.0) < 1e-14
    assert np.allclose(g[: 2 * rad + 1], g[2 * rad::-1])


# ---------------------------------------------------------------------------

def _sm(sf, shape, seed=77, bw=6):
    return sf.SmoothMedium(shape=shape, seed=seed, boundary_width=bw)


@pytest.mark.gpu
@pytest.mark.parametrize("shape", SHAPES + [(96, 130, 129)])
def test_gpu_generator_matches_port(port, shape):
    import paper_1609_03361_b200 as sf
    sm = _sm(sf, shape)
    lo, hi = sm.extrema()
    assert (lo, hi) == port.smooth_extrema(shape, 0, shape[0], 77)
    m, eta = sm.generate(lo, hi)
    pm, pe = port.smooth_medium(shape, 0, shape[0], 77, lo, hi, boundary_width=6)
    assert np.array_equal(bits(m), bits(pm))
    assert np.array_equal(bits(eta), bits(pe))
    # a slab of planes
    b, e = shape[0] // 4, shape[0] // 2 + 3
    ms, es = sm.generate(lo, hi, b, e)
    assert np.array_equal(bits(ms), bits(pm[b:e])) and np.array_equal(bits(es), bits(pe[b:e]))
    lb, hb = sm.extrema(b, e)
    assert (lb, hb) == port.smooth_extrema(shape, b, e, 77)


@pytest.mark.gpu
def test_gpu_generator_into_plan_and_slab_plans(port):
    """sf_plan_set_smooth_medium writes the plan's own planes: a whole-grid
    plan holds the global medium, slab plans their local planes (halos
    included), all bitwise the oracle's."""
    import ctypes as C

    import paper_1609_03361_b200 as sf
    from paper_1609_03361_b200 import _lib
    from paper_1609_03361_b200.slab import SlabPartition, SlabRun
    shape = (61, 40, 70)
    order, nt = 8, 4
    sm = _sm(sf, shape, seed=9, bw=5)
    lo, hi = sm.extrema()
    pm, pe = port.smooth_medium(shape, 0, shape[0], 9, lo, hi, boundary_width=5)
    model = sf.AcousticModel(shape=shape, boundary_width=5, spacing=10.0, nt=nt, space_order=order,
                             v_top=4500.0, v_bottom=4500.0)
    model.dt = 0.4 * 10.0 / 4500.0
    s = sf.acoustic_build(model, True)
    sm.set_plan(s.op, lo, hi)
    m = np.zeros(shape, np.float32)
    eta = np.zeros(shape, np.float32)
    s.op.download()
    assert np.array_equal(bits(s.m.data), bits(pm)) and np.array_equal(bits(s.eta.data), bits(pe))
    r = order // 2
    src = np.zeros((nt, 1), np.float32)
    ci, w = port.interp([[30 * 10.0, 20 * 10.0, 30 * 10.0]], 10.0, shape)
    for g in range(2):
        part = SlabPartition.split(shape[0], r, 2, g)
        sl = part.local()
        run = SlabRun(part, shape, order, True, nt, model.dt, 10.0, m[sl], eta[sl], src, ci, w,
                      np.zeros((nt, 1), np.float32), ci, w, local_medium=True)
        sf.api.check(_lib.lib.sf_plan_set_smooth_medium(run.plan, C.byref(sm.desc()), lo, hi))
        bufs = run.download()
        assert np.array_equal(bits(bufs[1]), bits(pm[sl]))
        assert np.array_equal(bits(bufs[2]), bits(pe[sl]))
        run.close()
    del m, eta


@pytest.mark.gpu
def test_gpu_generator_rejects_bad_input():
    import paper_1609_03361_b200 as sf
    sm = sf.SmoothMedium(shape=(20, 20, 20), sigma=100.0)
    with pytest.raises(sf.SfError):
        sm.extrema()
    sm = sf.SmoothMedium(shape=(20, 20, 20))
    with pytest.raises(sf.SfError):
        sm.extrema(5, 30)
    with pytest.raises(sf.SfError):
        sm.generate(1.0, 1.0)

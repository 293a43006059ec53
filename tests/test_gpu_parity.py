"""Parity of the CUDA path (through the C ABI) against the reference.

Bar: bitwise equality of every field slot and sparse trace with the
reference's generated kernel (the north-star tolerance is relative L2 1e-5
on fields and traces; the kernels reproduce the reference's fp32 operation
order, so equality is exact and asserted as such, with the 1e-5 relative L2
bound checked as well). The checker is the C restatement (oracle/sf_port.c),
itself pinned to the reference in test_oracle_pin.py, plus golden fixtures
made by the reference (tests/golden/).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a).view(np.uint32)


def rel_l2(a, b):
    a = a.astype(np.float64)
    b = b.astype(np.float64)
    n = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (n if n > 0 else 1.0)


def assert_parity(got, want):
    assert got.shape == want.shape
    assert rel_l2(got, want) <= 1e-5
    assert np.array_equal(bits(got), bits(want)), \
        f"not bitwise: max abs diff {np.abs(got.astype(np.float64) - want).max()}"


@pytest.fixture(scope="module")
def sf():
    import paper_1609_03361_b200 as sf
    if sf._lib.lib.sf_device_count() < 1:
        pytest.fail("no CUDA device: the GPU tests need a B200")
    return sf


def run_plan_raw(sf, shape, order, forward, dt, h, nt, m, eta, src, src_ci, src_w, rec, rec_ci,
                 rec_w, u=None):
    """Drive the raw C ABI (sf_acoustic_apply) with dense host buffers."""
    import ctypes as C
    from paper_1609_03361_b200 import _lib
    d = _lib.AcousticDesc()
    d.ndim = len(shape)
    for i, e in enumerate(shape):
        d.shape[i] = e
    d.space_order, d.forward, d.nt, d.dt, d.spacing = order, int(forward), nt, dt, h
    d.n_src, d.n_rec = src_ci.shape[0], rec_ci.shape[0]
    plan = C.c_void_p()
    sf.api.check(_lib.lib.sf_acoustic_plan_create(C.byref(d), 0, C.byref(plan)))
    try:
        u = np.zeros((3,) + tuple(shape), np.float32) if u is None else u
        bufs = [u, m, eta, src, src_ci, src_w, rec, rec_ci, rec_w]
        bufs = [np.ascontiguousarray(b) for b in bufs]
        rc = _lib.lib.sf_acoustic_apply(plan, *[b.ctypes.data for b in bufs])
        sf.api.check(rc)
        return bufs
    finally:
        _lib.lib.sf_plan_destroy(plan)


@pytest.mark.parametrize("tag", ["golden3d_fwd", "o8_3d_adj", "o4_2d_fwd"])
def test_golden_fields(sf, golden, tag):
    f = golden["fields"]
    nt, order, forward, dt, h = f[tag + "_meta"]
    nt, order, forward = int(nt), int(order), bool(forward)
    shape = f[tag + "_m"].shape
    src = f[tag + "_src"].copy() if forward else np.zeros_like(f[tag + "_src"])
    rec = np.zeros_like(f[tag + "_rec"]) if forward else f[tag + "_residual"].copy()
    out = run_plan_raw(sf, shape, order, forward, dt, h, nt, f[tag + "_m"], f[tag + "_eta"], src,
                       f[tag + "_src_ci"], f[tag + "_src_w"], rec, f[tag + "_rec_ci"],
                       f[tag + "_rec_w"])
    assert_parity(out[0], f[tag + "_field"])
    if forward:
        assert_parity(out[6], f[tag + "_rec"])
    else:
        assert_parity(out[3], f[tag + "_src"])


@pytest.mark.parametrize("tag", ["diff_o2", "diff_o4"])
def test_golden_diffusion(sf, golden, tag):
    from fractions import Fraction
    f = golden["fields"]
    n, nt, order, an, ad, dn, dd = (int(x) for x in f[tag + "_meta"])
    cfg = sf.DiffusionConfig(nx=n, ny=n, alpha=Fraction(an, ad), dx=Fraction(dn, dd),
                             dy=Fraction(dn, dd), nt=nt, order=order)
    b = sf.make_diffusion_operator(cfg)
    b.u.data[0] = f[tag + "_u0"]
    b.u.data[1] = f[tag + "_u0"]
    b.op.apply()
    assert_parity(b.u.data, f[tag + "_out"])


def random_case(port, shape, order, seed, nsrc=3, nrec=17, spacing=10.0):
    rng = np.random.default_rng(seed)
    nd = len(shape)
    v = 1500.0 + 3000.0 * rng.random(shape)
    m, eta = port.medium_from_velocity(v, 5, spacing, 1500.0)
    dt = min(0.4 * spacing / 4500.0, port.stable_dt(nd, order, spacing, 4500.0, 4500.0))
    lo = (order // 2 + 1) * spacing
    def pts(n):
        return np.stack([rng.uniform(lo, (e - order // 2 - 2) * spacing, n) for e in shape], 1)
    src_c, rec_c = pts(nsrc), pts(nrec)
    if nsrc >= 2:  # force a collision: two sources in the same cell
        src_c[1] = src_c[0] + 0.1 * spacing * rng.random(nd)
    if nrec >= 2:
        rec_c[1] = rec_c[0] + 0.2 * spacing * rng.random(nd)
    src_ci, src_w = port.interp(src_c, spacing, shape)
    rec_ci, rec_w = port.interp(rec_c, spacing, shape)
    return dict(m=m, eta=eta, dt=dt, src_ci=src_ci, src_w=src_w, rec_ci=rec_ci, rec_w=rec_w,
                rng=rng)


@pytest.mark.parametrize("order", [2, 4, 6, 8, 10, 12, 14, 16])
@pytest.mark.parametrize("forward", [True, False])
def test_acoustic3d_random_medium_vs_oracle(sf, port, order, forward):
    shape = (37, 45, 70)  # ragged: 70 is not a multiple of 32, 45 not of 16
    nt = 23
    c = random_case(port, shape, order, seed=order * 7 + forward)
    rng = c["rng"]
    series_src = rng.standard_normal((nt, 3)).astype(np.float32)
    series_rec = rng.standard_normal((nt, 17)).astype(np.float32)
    u0 = (1e-3 * rng.standard_normal((3,) + shape)).astype(np.float32)
    if forward:
        src, rec = series_src, np.zeros((nt, 17), np.float32)
    else:
        src, rec = np.zeros((nt, 3), np.float32), series_rec
    out = run_plan_raw(sf, shape, order, forward, c["dt"], 10.0, nt, c["m"], c["eta"], src.copy(),
                       c["src_ci"], c["src_w"], rec.copy(), c["rec_ci"], c["rec_w"], u=u0.copy())
    coefs = port.coefs(3, order, forward, c["dt"], 10.0)
    u = u0.copy()
    if forward:
        port.acoustic_run(coefs, u, c["m"], c["eta"], src, c["src_ci"], c["src_w"], rec,
                          c["rec_ci"], c["rec_w"], nt)
        assert_parity(out[6], rec)
    else:
        port.acoustic_run(coefs, u, c["m"], c["eta"], rec, c["rec_ci"], c["rec_w"], src,
                          c["src_ci"], c["src_w"], nt)
        assert_parity(out[3], src)
    assert_parity(out[0], u)


@pytest.mark.parametrize("order", [2, 8, 16])
@pytest.mark.parametrize("forward", [True, False])
def test_acoustic2d_vs_oracle(sf, port, order, forward):
    shape = (61, 83)
    nt = 40
    c = random_case(port, shape, order, seed=100 + order)
    rng = c["rng"]
    src = rng.standard_normal((nt, 3)).astype(np.float32) if forward else np.zeros((nt, 3), np.float32)
    rec = np.zeros((nt, 17), np.float32) if forward else rng.standard_normal((nt, 17)).astype(np.float32)
    out = run_plan_raw(sf, shape, order, forward, c["dt"], 10.0, nt, c["m"], c["eta"], src.copy(),
                       c["src_ci"], c["src_w"], rec.copy(), c["rec_ci"], c["rec_w"])
    coefs = port.coefs(2, order, forward, c["dt"], 10.0)
    u = np.zeros((3,) + shape, np.float32)
    if forward:
        port.acoustic_run(coefs, u, c["m"], c["eta"], src, c["src_ci"], c["src_w"], rec,
                          c["rec_ci"], c["rec_w"], nt)
        assert_parity(out[6], rec)
    else:
        port.acoustic_run(coefs, u, c["m"], c["eta"], rec, c["rec_ci"], c["rec_w"], src,
                          c["src_ci"], c["src_w"], nt)
        assert_parity(out[3], src)
    assert_parity(out[0], u)


def test_api_forward_matches_live_reference(sf, ref):
    """acoustic_forward through the mirrored API vs the reference's own
    acoustic_build + Operator::apply on the same default model."""
    from oracle_lib import AcousticCase, ref_acoustic
    model = sf.AcousticModel(shape=(48, 40, 36), nt=40, boundary_width=6, spacing=10.0,
                             space_order=8)
    s = sf.acoustic_forward(model)
    op = ref_acoustic(ref, AcousticCase(shape=(48, 40, 36), nt=40, boundary_width=6,
                                        spacing=10.0, space_order=8), True)
    op.apply()
    assert_parity(s.field.data, op.get("u", np.float32, (3, 48, 40, 36)))
    assert_parity(s.rec.data.data, op.get("rec", np.float32, (40, 8)))


def test_zero_steps_is_identity(sf):
    # test_codegen.cpp:127-135: nt = 0 leaves the buffers unchanged
    cfg = sf.DiffusionConfig(nx=16, ny=16, nt=0)
    u0 = sf.gaussian_blob_field(16, 16)
    out = sf.diffusion_run(cfg, u0)
    assert np.array_equal(out, u0.astype(np.float32).astype(np.float64))
    # an acoustic model with nt = 0 has empty sparse series: rejected like
    # the reference's create_array (grid.cpp:179-188)
    with pytest.raises(sf.InvalidShapeError):
        sf.acoustic_build(sf.AcousticModel(shape=(24, 24, 20), nt=0, boundary_width=4), True)


def test_zero_source_zero_field(sf):
    model = sf.AcousticModel(shape=(30, 30, 30), nt=20, boundary_width=4)
    s = sf.acoustic_forward(model, np.zeros(20))
    assert not s.field.data.any() and not s.rec.data.data.any()


def test_signature_mismatch(sf):
    model = sf.AcousticModel(shape=(24, 24, 20), nt=2, boundary_width=4)
    s = sf.acoustic_build(model, True)
    with pytest.raises(sf.SignatureMismatchError):
        s.op.apply([s.m] + s.op.args[1:])
    with pytest.raises(sf.SignatureMismatchError):
        s.op.apply(s.op.args[:-1])


def test_adjoint_dot_test(sf):
    """Acceptance criterion 5 (acceptance.cpp:208-245) on the GPU path."""
    for order in (2, 4, 6, 8, 10, 12):
        m = sf.AcousticModel(shape=(60, 60), nt=250, boundary_width=10, space_order=order)
        r = sf.adjoint_test(m, 7)
        assert not r.degenerate and abs(r.ratio - 1.0) <= 1e-5, (order, r)
    for order in (2, 4):
        m = sf.AcousticModel(shape=(40, 40, 30), nt=120, boundary_width=8, space_order=order)
        r = sf.adjoint_test(m, 11)
        assert not r.degenerate and abs(r.ratio - 1.0) <= 1e-5, (order, r)


def test_adjoint_dot_test_matches_reference_products(sf, ref):
    import ctypes as C
    ref.lib.sfref_adjoint_test.argtypes = [C.c_int, np.ctypeslib.ndpointer(np.int64), C.c_int,
                                           C.c_double, C.c_long, C.c_int, C.c_uint,
                                           np.ctypeslib.ndpointer(np.float64)]
    out = np.zeros(4)
    assert ref.lib.sfref_adjoint_test(2, np.array([60, 60], np.int64), 10, 15.0, 100, 4, 7,
                                      out) == 0
    r = sf.adjoint_test(sf.AcousticModel(shape=(60, 60), nt=100, boundary_width=10,
                                         space_order=4), 7)
    assert r.forward_product == out[0] and r.adjoint_product == out[1]


def test_diffusion_config1_layout_and_oracle(sf, port):
    """Config 1 at full size (2048^2, order 2, exact 1/4 weights) vs the
    port, bitwise, on a reduced step count."""
    from fractions import Fraction
    n, nt = 2048, 60
    rng = np.random.default_rng(1)
    u0 = np.zeros((n, n), np.float32)
    u0[1:-1, 1:-1] = rng.random((n - 2, n - 2))
    cfg = sf.DiffusionConfig(nx=n, ny=n, alpha=Fraction(1, 2), dx=Fraction(1, 2047),
                             dy=Fraction(1, 2047), nt=nt, order=2)
    assert cfg.dt() == Fraction(1, 8380418)
    b = sf.make_diffusion_operator(cfg)
    b.u.data[0] = u0
    b.u.data[1] = u0
    b.op.apply()
    u = np.stack([u0, u0])
    port.diffusion_run(u, 2, (1, 2), (1, 2047), nt)
    assert_parity(b.u.data, u)


@pytest.mark.parametrize("warps", ["default", "16"])
def test_fwi_gradient_vs_oracle(sf, port, monkeypatch, warps):
    if warps != "default":  # forward sweep on 64 x 32 tiles
        monkeypatch.setenv("SF_VEC_WARPS", warps)
    shape = (34, 30, 40)
    order, nt = 8, 25
    c = random_case(port, shape, order, seed=5, nsrc=1, nrec=40)
    rng = c["rng"]
    src = rng.standard_normal((nt, 1)).astype(np.float32)
    residual = rng.standard_normal((nt, 40)).astype(np.float32)
    plan = sf.FwiPlan(shape, order, nt, c["dt"], 10.0, 1, 40)
    rec_out, grad, v, srcs = plan.gradient(c["m"], c["eta"], src, c["src_ci"], c["src_w"],
                                           c["rec_ci"], c["rec_w"], residual, want_v=True,
                                           want_src=True)
    cf = port.coefs(3, order, True, c["dt"], 10.0)
    hist = np.zeros((nt + 2,) + shape, np.float32)
    rec = np.zeros((nt, 40), np.float32)
    port.forward_history(cf, hist, c["m"], c["eta"], src, c["src_ci"], c["src_w"], rec,
                         c["rec_ci"], c["rec_w"], nt)
    assert_parity(rec_out, rec)
    # the history run is bitwise the 3-slot forward
    u = np.zeros((3,) + shape, np.float32)
    rec2 = np.zeros_like(rec)
    port.acoustic_run(cf, u, c["m"], c["eta"], src, c["src_ci"], c["src_w"], rec2, c["rec_ci"],
                      c["rec_w"], nt)
    assert np.array_equal(bits(hist[nt + 1]), bits(u[nt % 3]))
    ca = port.coefs(3, order, False, c["dt"], 10.0)
    vv = np.zeros((3,) + shape, np.float32)
    g = np.zeros(shape, np.float32)
    s2 = np.zeros((nt, 1), np.float32)
    port.adjoint_gradient(ca, vv, c["m"], c["eta"], hist, residual, c["rec_ci"], c["rec_w"], s2,
                          c["src_ci"], c["src_w"], g, nt)
    assert_parity(v, vv)
    assert_parity(srcs, s2)
    assert np.abs(g).max() > 0
    assert_parity(grad, g)


@pytest.mark.parametrize("order,n,nt", [(2, 203, 37), (4, 150, 19), (8, 97, 13), (16, 70, 5)])
def test_diffusion_temporal_blocking_vs_oracle(sf, port, order, n, nt):
    """Temporally blocked diffusion (several steps per launch) vs the port:
    ragged grids, step counts that are not multiples of the block depth, and
    slots whose boundary strips differ (each level must see its own slot's
    boundary values, as in the reference's 2-slot loop)."""
    from fractions import Fraction
    rng = np.random.default_rng(order)
    u = rng.random((2, n, n)).astype(np.float32)
    cfg = sf.DiffusionConfig(nx=n, ny=n, alpha=Fraction(1, 3), dx=Fraction(1, n - 1),
                             dy=Fraction(1, n - 1), nt=nt, order=order)
    b = sf.make_diffusion_operator(cfg)
    b.u.data[...] = u
    b.op.apply()
    ref = u.copy()
    port.diffusion_run(ref, order, (1, 3), (1, n - 1), nt)
    assert_parity(b.u.data, ref)


@pytest.mark.parametrize("tile,rv", [("48", "1"), ("56", "1"), ("64", "1"), ("64", "2"),
                                     ("72", "1"), ("80", "1"), ("96", "1")])
def test_diffusion_tile_variants_vs_oracle(sf, port, monkeypatch, tile, rv):
    """Radius-1 temporal blocking with every selectable core tile
    (SF_TB_TILE; 64 is the measured default) and one or two rows per thread
    visit (SF_TB_RV; 2 is the default) on a ragged grid."""
    from fractions import Fraction
    monkeypatch.setenv("SF_TB_TILE", tile)
    monkeypatch.setenv("SF_TB_RV", rv)
    n, nt = 301, 21
    rng = np.random.default_rng(int(tile))
    u = rng.random((2, n, n)).astype(np.float32)
    cfg = sf.DiffusionConfig(nx=n, ny=n, alpha=Fraction(1, 3), dx=Fraction(1, n - 1),
                             dy=Fraction(1, n - 1), nt=nt, order=2)
    b = sf.make_diffusion_operator(cfg)
    b.u.data[...] = u
    b.op.apply()
    ref = u.copy()
    port.diffusion_run(ref, 2, (1, 3), (1, n - 1), nt)
    assert_parity(b.u.data, ref)


VARIANTS = [{}, {"SF_VEC": "0"}, {"SF_NO_TMA": "1"}, {"SF_VEC": "0", "SF_TMA": "1"},
            {"SF_VECQ": "0"}, {"SF_VEC_WARPS": "8"}, {"SF_TMA_STAGES": "2"},
            {"SF_VEC": "0", "SF_NO_TMA": "1", "SF_TILE": "2,16"}, {"SF_VEC_NX": "1"},
            {"SF_VEC_NX": "1", "SF_TMA_STAGES": "4"}, {"SF_NO_FUSED_SPARSE": "1"},
            {"SF_VEC_RPL": "2"}, {"SF_VEC_RPL": "2", "SF_VEC_NX": "1"},
            {"SF_VEC_RPL": "2", "SF_VEC_NX": "2", "SF_VEC_WARPS": "8"}, {"SF_VECQ2": "1"},
            {"SF_VECQ2": "1", "SF_TMA_STAGES": "3"}, {"SF_VECQ_FORM": "free"},
            {"SF_VECQ_FORM": "pinned"}, {"SF_VECQ_FORM": "tmem"}, {"SF_VEC_WARPS": "16"},
            {"SF_VEC_NX": "1", "SF_VEC_WARPS": "8"}, {"SF_VEC_WARPS": "16", "SF_VEC_AQ": "1"}, {"SF_VEC_WARPS": "16", "SF_VEC_AQ": "0"},
            {"SF_VEC_WARPS": "8", "SF_VEC_AQ8": "1"}, {"SF_VEC_WARPS": "16", "SF_VEC_AQ2": "1"},
            {"SF_VEC_WARPS": "16", "SF_VEC_AQ2": "1", "SF_ZCHUNKS": "3"},
            {"SF_VECQ_FORM": "last"}, {"SF_VEC_WARPS": "8", "SF_VECQ_FORM": "last"},
            {"SF_VEC_WARPS": "12"}, {"SF_VEC_WARPS": "12", "SF_VECQ_FORM": "last"}]


@pytest.mark.parametrize("order", [2, 6, 8, 12, 16])
@pytest.mark.parametrize("env", VARIANTS, ids=lambda e: ",".join(f"{k}={v}" for k, v in e.items()) or "default")
def test_every_kernel_variant_bitwise(sf, port, monkeypatch, order, env):
    """Each stencil kernel family (per-thread loads, scalar TMA, vector TMA
    ring, queue-vector TMA), tile and pipeline depth reproduces the oracle."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    shape = (29, 37, 101)
    nt = 9
    c = random_case(port, shape, order, seed=order + 31)
    rng = c["rng"]
    src = rng.standard_normal((nt, 3)).astype(np.float32)
    rec = np.zeros((nt, 17), np.float32)
    out = run_plan_raw(sf, shape, order, True, c["dt"], 10.0, nt, c["m"], c["eta"], src.copy(),
                       c["src_ci"], c["src_w"], rec.copy(), c["rec_ci"], c["rec_w"])
    coefs = port.coefs(3, order, True, c["dt"], 10.0)
    u = np.zeros((3,) + shape, np.float32)
    port.acoustic_run(coefs, u, c["m"], c["eta"], src, c["src_ci"], c["src_w"], rec, c["rec_ci"],
                      c["rec_w"], nt)
    assert_parity(out[0], u)
    assert_parity(out[6], rec)


@pytest.mark.parametrize("order", [10, 12, 14, 16])
@pytest.mark.parametrize("zchunks", ["1", "3"])
@pytest.mark.parametrize("form", ["default", "tmem", "last"])
def test_queue_kernel_long_chunks(sf, port, monkeypatch, order, zchunks, form):
    """The queue-vector kernel over a-0 chunks long enough for every pipeline
    stage to be refilled many times and the register queue to cycle through
    many two-step passes (or, in the TMEM form, the window to be moved back
    to slot 0 several times), odd and even chunk lengths: bitwise the
    oracle."""
    monkeypatch.setenv("SF_ZCHUNKS", zchunks)
    if form != "default":
        monkeypatch.setenv("SF_VECQ_FORM", form)
    shape = (97, 30, 77)
    nt = 4
    c = random_case(port, shape, order, seed=order + 7)
    rng = c["rng"]
    src = rng.standard_normal((nt, 3)).astype(np.float32)
    rec = np.zeros((nt, 17), np.float32)
    out = run_plan_raw(sf, shape, order, True, c["dt"], 10.0, nt, c["m"], c["eta"], src.copy(),
                       c["src_ci"], c["src_w"], rec.copy(), c["rec_ci"], c["rec_w"])
    coefs = port.coefs(3, order, True, c["dt"], 10.0)
    u = np.zeros((3,) + shape, np.float32)
    port.acoustic_run(coefs, u, c["m"], c["eta"], src, c["src_ci"], c["src_w"], rec, c["rec_ci"],
                      c["rec_w"], nt)
    assert_parity(out[0], u)
    assert_parity(out[6], rec)


@pytest.mark.parametrize("order", [4, 12])
def test_autotune_then_parity(sf, port, order):
    """Operator::autotune on the GPU: every candidate is timed, the best is
    kept, the state is restored, and the tuned plan still matches the oracle."""
    model = sf.AcousticModel(shape=(40, 44, 70), nt=12, boundary_width=5, spacing=10.0,
                             space_order=order)
    s = sf.acoustic_build(model, True)
    s.op.upload()
    report, best = s.op.autotune(tune_nt=4, repeats=1)
    assert len(report) >= 4 and best is not None
    assert all(t > 0 for _, t in report)
    s.op.apply()
    c = port.coefs(3, order, True, s.dt, 10.0)
    u = np.zeros_like(s.field.data)
    rec = np.zeros_like(s.rec.data.data)
    port.acoustic_run(c, u, s.m.data, s.eta.data, s.src.data.data.copy(), s.src.ci.data,
                      s.src.w.data, rec, s.rec.ci.data, s.rec.w.data, model.nt)
    assert_parity(s.field.data, u)
    assert_parity(s.rec.data.data, rec)


def test_hbm_buffer_io_interchanges_with_reference(sf, ref, tmp_path):
    """save_buffer/load_buffer from HBM in the reference's SFG1 format: files
    written from the device load into the reference and vice versa."""
    import ctypes as C
    from oracle_lib import AcousticCase, ref_acoustic
    ref.lib.sfref_save_buffer.argtypes = [C.c_void_p, C.c_char_p, C.c_char_p]
    ref.lib.sfref_load_buffer.argtypes = [C.c_void_p, C.c_char_p, C.c_char_p]
    model = sf.AcousticModel(shape=(24, 24, 20), nt=12, boundary_width=4)
    s = sf.acoustic_forward(model)
    op = ref_acoustic(ref, AcousticCase(shape=(24, 24, 20), nt=12, boundary_width=4), True)
    for name, dt, shape in [("u", np.float32, (3, 24, 24, 20)), ("rec", np.float32, (12, 8)),
                            ("src_ci", np.int32, (1, 3)), ("m", np.float32, (24, 24, 20))]:
        path = str(tmp_path / f"{name}.sfg")
        s.op.save_buffer(name, path)
        assert ref.lib.sfref_load_buffer(op.h, name.encode(), path.encode()) == 0, ref.error()
        want = {"u": s.field.data, "rec": s.rec.data.data, "src_ci": s.src.ci.data,
                "m": s.m.data}[name]
        assert np.array_equal(op.get(name, dt, shape), want)
    # reference -> device
    op.apply()
    path = str(tmp_path / "u_ref.sfg")
    assert ref.lib.sfref_save_buffer(op.h, b"u", path.encode()) == 0
    s.op.load_buffer("u", path)
    s.op.download()
    assert np.array_equal(bits(s.field.data), bits(op.get("u", np.float32, (3, 24, 24, 20))))
    with pytest.raises(sf.SfError):
        s.op.load_buffer("m", path)  # shape/rank mismatch is rejected


def test_text_dumps_match_reference(sf, ref, tmp_path):
    """dump_csv (grid.cpp:256-273) and save_series_text (sparse.cpp:215-227)
    from HBM are byte-identical to the reference's own files; the series
    reader load_series_column (sparse.cpp:205-213) reads them back alike."""
    import ctypes as C
    from oracle_lib import AcousticCase, ref_acoustic, ref_diffusion
    ref.lib.sfref_dump_csv.argtypes = [C.c_void_p, C.c_char_p, C.c_char_p, C.c_long]
    ref.lib.sfref_save_series_text.argtypes = [C.c_void_p, C.c_char_p, C.c_char_p]
    ref.lib.sfref_load_series_column.restype = C.c_long
    ref.lib.sfref_load_series_column.argtypes = [C.c_char_p, C.c_void_p, C.c_long]
    model = sf.AcousticModel(shape=(48, 44), nt=60, boundary_width=6, spacing=10.0,
                             space_order=4)
    s = sf.acoustic_forward(model)
    op = ref_acoustic(ref, AcousticCase(shape=(48, 44), nt=60, boundary_width=6,
                                        spacing=10.0, space_order=4), True)
    op.apply()
    files = []
    for name, slot in [("u", 0), ("u", 1), ("u", 2), ("m", 0), ("eta", 0)]:
        mine, theirs = tmp_path / f"{name}{slot}.csv", tmp_path / f"{name}{slot}_ref.csv"
        s.op.dump_csv(name, mine, slot)
        assert ref.lib.sfref_dump_csv(op.h, name.encode(), str(theirs).encode(), slot) == 0
        files.append((mine, theirs))
    for name in ("rec", "src"):
        mine, theirs = tmp_path / f"{name}.txt", tmp_path / f"{name}_ref.txt"
        s.op.save_series_text(name, mine)
        assert ref.lib.sfref_save_series_text(op.h, name.encode(), str(theirs).encode()) == 0
        files.append((mine, theirs))
    for mine, theirs in files:
        assert mine.read_bytes() == theirs.read_bytes(), mine.name
    # the reader: same numbers as the reference's parser
    path = files[-2][0]
    got = sf.load_series_column(path)
    want = np.zeros(got.size + 8)
    n = ref.lib.sfref_load_series_column(str(path).encode(), want.ctypes.data, want.size)
    assert n == got.size and np.array_equal(got, want[:n])
    # diffusion (time-varying, 2 slots) and the rejections
    d = sf.make_diffusion_operator(sf.DiffusionConfig(nx=40, ny=36, nt=7))
    d.u.data[...] = np.random.default_rng(3).random(d.u.data.shape, dtype=np.float32)
    d.op.apply()
    rop = ref_diffusion(ref, 40, 36, (1, 2), (1, 39), 7, 2)
    rop.set("u", d.u.data)
    for slot in (0, 1):
        mine, theirs = tmp_path / f"d{slot}.csv", tmp_path / f"d{slot}_ref.csv"
        d.op.dump_csv("u", mine, slot)
        assert ref.lib.sfref_dump_csv(rop.h, b"u", str(theirs).encode(), slot) == 0
        assert mine.read_bytes() == theirs.read_bytes()
    with pytest.raises(sf.SfError):
        d.op.dump_csv("u", tmp_path / "bad.csv", 2)
    s3 = sf.acoustic_forward(sf.AcousticModel(shape=(24, 24, 20), nt=5, boundary_width=4))
    with pytest.raises(sf.SfError):
        s3.op.dump_csv("u", tmp_path / "bad3d.csv", 0)   # 2D grids only
    with pytest.raises(sf.SfError):
        s3.op.save_series_text("m", tmp_path / "bad.txt")


def test_reciprocal_exact_on_every_float(sf):
    """The stencil kernels' batched reciprocal (fast path + guarded library
    fallback) equals __frcp_rn == __fdiv_rn(1, x) on all 2^32 inputs."""
    import ctypes as C
    bad = C.c_ulonglong(123)
    assert sf._lib.lib.sf_selftest_reciprocal(0, C.byref(bad)) == 0, sf._lib.last_error()
    assert bad.value == 0


@pytest.mark.parametrize("order,shape", [(4, (30, 41, 75)), (4, (26, 38, 101)), (8, (34, 40, 70)),
                                         (2, (22, 27, 45))])
@pytest.mark.parametrize("forward", [True, False])
@pytest.mark.parametrize("split", [None, (1, 5), (3, 4, 9)])
def test_step_ranges_and_tile_edge_points(sf, port, order, shape, forward, split):
    """The fused sparse epilogue (injection per CTA tile, sampling one step
    late) under every way of cutting [0, nt) into sf_plan_run ranges, with
    points on tile edges, sharing cells, and one in the non-interior shell
    (which turns the fused path off for the plan)."""
    import ctypes as C
    from paper_1609_03361_b200 import _lib
    nt = 11
    r = order // 2
    h = 10.0
    rng = np.random.default_rng(order * 100 + shape[2] + int(forward))
    v = 1500.0 + 3000.0 * rng.random(shape)
    m, eta = port.medium_from_velocity(v, 4, h, 1500.0)
    dt = min(0.4 * h / 4500.0, port.stable_dt(3, order, h, 4500.0, 4500.0))
    # cells on 32- and 64-wide tile edges in a2, 8/16-row edges in a1, chunk
    # edges in a0, a shared cell, plus (maybe) one point in the outer shell
    cells = [(r + 1, 15.5, 31.5), (shape[0] // 2, 16.0, 32.0), (shape[0] - r - 2, 7.5, 63.5),
             (r + 3, 8.2, 31.9), (r + 3, 8.2, 31.9)]
    inner = [[a0 * h, a1 * h, min(a2, shape[2] - r - 2.5) * h] for a0, a1, a2 in cells]
    rec_c = np.concatenate([inner, np.stack([rng.uniform((r + 1) * h, (e - r - 2) * h, 37)
                                             for e in shape], 1)])
    src_c = np.array(inner[:4] + ([[0.3 * h, 9.0 * h, 9.0 * h]] if split == (1, 5) else []))
    src_ci, src_w = port.interp(src_c, h, shape)
    rec_ci, rec_w = port.interp(rec_c, h, shape)
    ns, nr = len(src_ci), len(rec_ci)
    u0 = (1e-3 * rng.standard_normal((3,) + shape)).astype(np.float32)
    if forward:
        src = rng.standard_normal((nt, ns)).astype(np.float32)
        rec = np.zeros((nt, nr), np.float32)
    else:
        src = np.zeros((nt, ns), np.float32)
        rec = rng.standard_normal((nt, nr)).astype(np.float32)
    # oracle
    coefs = port.coefs(3, order, forward, dt, h)
    want_u, want_src, want_rec = u0.copy(), src.copy(), rec.copy()
    if forward:
        port.acoustic_run(coefs, want_u, m, eta, want_src, src_ci, src_w, want_rec, rec_ci, rec_w, nt)
    else:
        port.acoustic_run(coefs, want_u, m, eta, want_rec, rec_ci, rec_w, want_src, src_ci, src_w,
                          nt)
    # GPU, in pieces
    d = _lib.AcousticDesc()
    d.ndim = 3
    for i, e in enumerate(shape):
        d.shape[i] = e
    d.space_order, d.forward, d.nt, d.dt, d.spacing = order, int(forward), nt, dt, h
    d.n_src, d.n_rec = ns, nr
    plan = C.c_void_p()
    sf.api.check(_lib.lib.sf_acoustic_plan_create(C.byref(d), 0, C.byref(plan)))
    try:
        bufs = [np.ascontiguousarray(b) for b in
                (u0.copy(), m, eta, src.copy(), src_ci, src_w, rec.copy(), rec_ci, rec_w)]
        argv = (C.c_void_p * 9)(*[b.ctypes.data for b in bufs])
        sf.api.check(_lib.lib.sf_plan_upload(plan, argv, 9))
        edges = [0] + list(split or []) + [nt]
        for a, b in zip(edges[:-1], edges[1:]):
            sf.api.check(_lib.lib.sf_plan_run(plan, a, b))
        sf.api.check(_lib.lib.sf_plan_download(plan, argv, 9))
    finally:
        _lib.lib.sf_plan_destroy(plan)
    assert_parity(bufs[0], want_u)
    assert_parity(bufs[6] if forward else bufs[3], want_rec if forward else want_src)


@pytest.mark.parametrize("shape,order,ns,nr,nt", [
    ((9, 9, 9), 8, 1, 1, 1),        # interior of a single point per axis
    ((10, 40, 70), 8, 0, 3, 4),     # no sources
    ((30, 20, 33), 4, 2, 0, 5),     # no receivers
    ((18, 17, 130), 16, 1, 2, 3),   # order 16 on a thin grid
    ((6, 7, 5), 2, 3, 3, 6),        # tiny grid, order 2
])
@pytest.mark.parametrize("forward", [True, False])
def test_degenerate_shapes_and_empty_point_sets(sf, port, shape, order, ns, nr, nt, forward):
    rng = np.random.default_rng(sum(shape) + order)
    h = 10.0
    r = order // 2
    v = 1500.0 + 3000.0 * rng.random(shape)
    m, eta = port.medium_from_velocity(v, 2, h, 1500.0)
    dt = min(0.4 * h / 4500.0, port.stable_dt(3, order, h, 4500.0, 4500.0))

    def pts(n):
        if n == 0:
            return np.zeros((0, 3), np.int32), np.zeros((0, 8), np.float32)
        c = np.stack([rng.uniform(0.2 * h, (e - 1.2) * h, n) for e in shape], 1)
        return port.interp(c, h, shape)
    src_ci, src_w = pts(ns)
    rec_ci, rec_w = pts(nr)
    u0 = (1e-3 * rng.standard_normal((3,) + shape)).astype(np.float32)
    src = (rng.standard_normal((nt, ns)) if forward else np.zeros((nt, ns))).astype(np.float32)
    rec = (np.zeros((nt, nr)) if forward else rng.standard_normal((nt, nr))).astype(np.float32)
    if ns == 0 or nr == 0:
        # a zero-extent sparse series is rejected, as the reference's
        # create_array rejects it (grid.cpp:179-188)
        with pytest.raises(sf.InvalidShapeError):
            run_plan_raw(sf, shape, order, forward, dt, h, nt, m, eta, src, src_ci, src_w, rec,
                         rec_ci, rec_w, u=u0.copy())
        return
    out = run_plan_raw(sf, shape, order, forward, dt, h, nt, m, eta, src.copy(), src_ci, src_w,
                       rec.copy(), rec_ci, rec_w, u=u0.copy())
    coefs = port.coefs(3, order, forward, dt, h)
    u = u0.copy()
    if forward:
        port.acoustic_run(coefs, u, m, eta, src, src_ci, src_w, rec, rec_ci, rec_w, nt)
        assert_parity(out[6], rec)
    else:
        port.acoustic_run(coefs, u, m, eta, rec, rec_ci, rec_w, src, src_ci, src_w, nt)
        assert_parity(out[3], src)
    assert_parity(out[0], u)


@pytest.mark.parametrize("order", [4, 8, 12])
def test_eta_zero_boxes_skipped_bitwise(sf, port, order):
    """The vector kernels skip the TMA load of eta boxes that are all +0.0
    and use 0.0f instead. Boxes holding -0.0, a single nonzero value, or
    whose content changes between two applies of one plan (the flags are
    recomputed when eta is re-uploaded) must still be read."""
    import ctypes as C
    from paper_1609_03361_b200 import _lib
    shape = (44, 53, 100)
    nt = 9
    c = random_case(port, shape, order, seed=100 + order)
    rng = c["rng"]
    eta1 = np.zeros(shape, np.float32)
    eta1[:6] = c["eta"][:6]             # damped top planes only
    eta1[20, 30, 70] = 3.0e-4            # one nonzero value inside a box
    eta1[25, 10:14, 40:44] = -0.0        # negative zeros: not skippable
    eta2 = c["eta"].copy()               # second apply: the full sponge
    eta2[30, 20, 50] = -0.0
    d = _lib.AcousticDesc()
    d.ndim = 3
    for i, e in enumerate(shape):
        d.shape[i] = e
    d.space_order, d.forward, d.nt, d.dt, d.spacing = order, 1, nt, c["dt"], 10.0
    d.n_src, d.n_rec = c["src_ci"].shape[0], c["rec_ci"].shape[0]
    plan = C.c_void_p()
    sf.api.check(_lib.lib.sf_acoustic_plan_create(C.byref(d), 0, C.byref(plan)))
    coefs = port.coefs(3, order, True, c["dt"], 10.0)
    try:
        fractions = []
        for eta in (eta1, eta2):
            src = rng.standard_normal((nt, 3)).astype(np.float32)
            u0 = (1e-3 * rng.standard_normal((3,) + shape)).astype(np.float32)
            bufs = [u0.copy(), c["m"], eta, src.copy(), c["src_ci"], c["src_w"],
                    np.zeros((nt, 17), np.float32), c["rec_ci"], c["rec_w"]]
            bufs = [np.ascontiguousarray(b) for b in bufs]
            sf.api.check(_lib.lib.sf_acoustic_apply(plan, *[b.ctypes.data for b in bufs]))
            frac = C.c_double()
            sf.api.check(_lib.lib.sf_plan_eta_skip_fraction(plan, C.byref(frac)))
            fractions.append(frac.value)
            u = u0.copy()
            rec = np.zeros((nt, 17), np.float32)
            port.acoustic_run(coefs, u, c["m"], eta, src, c["src_ci"], c["src_w"], rec,
                              c["rec_ci"], c["rec_w"], nt)
            assert_parity(bufs[0], u)
            assert_parity(bufs[6], rec)
        assert fractions[0] > 0.5          # most boxes of eta1 are +0.0
        assert fractions[1] < fractions[0]  # the sponge leaves fewer
    finally:
        _lib.lib.sf_plan_destroy(plan)


@pytest.mark.parametrize("order", [4, 8, 16])
@pytest.mark.parametrize("forward", [True, False])
def test_special_values_bitwise(sf, port, order, forward):
    """Signed zeros, subnormals and near-limit magnitudes in the wavefield,
    tiny m (reciprocals on the slow path) and subnormal eta: the kernels keep
    IEEE semantics (no flush-to-zero, no contraction), so the result is still
    bitwise the CPU oracle's. (NaN is excluded: its payload is not specified
    by IEEE and differs between x86 and the GPU.)"""
    shape = (30, 38, 70)
    nt = 7
    c = random_case(port, shape, order, seed=500 + order + forward)
    rng = c["rng"]
    u0 = (1e-3 * rng.standard_normal((3,) + shape)).astype(np.float32)
    pick = rng.random((3,) + shape)
    u0[pick < 0.15] = 0.0
    u0[(pick >= 0.15) & (pick < 0.3)] = -0.0
    sub = (pick >= 0.3) & (pick < 0.45)
    u0[sub] = (rng.standard_normal(sub.sum()) * 1e-39).astype(np.float32)  # subnormals
    big = (pick >= 0.45) & (pick < 0.47)
    u0[big] = (rng.standard_normal(big.sum()) * 1e30).astype(np.float32)
    m = c["m"].copy()
    mp = rng.random(shape)
    m[mp < 0.05] = 1e-30                       # t3 near the float range: slow reciprocal path
    eta = c["eta"].copy()
    eta[(mp >= 0.05) & (mp < 0.1)] = 1e-40     # subnormal damping
    eta[(mp >= 0.1) & (mp < 0.15)] = -0.0
    assert np.isfinite(u0).all()
    src = rng.standard_normal((nt, 3)).astype(np.float32)
    rec = rng.standard_normal((nt, 17)).astype(np.float32)
    if forward:
        s_in, r_in = src, np.zeros_like(rec)
    else:
        s_in, r_in = np.zeros_like(src), rec
    out = run_plan_raw(sf, shape, order, forward, c["dt"], 10.0, nt, m, eta, s_in.copy(),
                       c["src_ci"], c["src_w"], r_in.copy(), c["rec_ci"], c["rec_w"], u=u0.copy())
    coefs = port.coefs(3, order, forward, c["dt"], 10.0)
    u = u0.copy()
    if forward:
        r = r_in.copy()
        port.acoustic_run(coefs, u, m, eta, s_in.copy(), c["src_ci"], c["src_w"], r, c["rec_ci"],
                          c["rec_w"], nt)
        got_tr, want_tr = out[6], r
    else:
        s = s_in.copy()
        port.acoustic_run(coefs, u, m, eta, r_in.copy(), c["rec_ci"], c["rec_w"], s, c["src_ci"],
                          c["src_w"], nt)
        got_tr, want_tr = out[3], s
    fin = np.isfinite(u)
    assert np.array_equal(np.isfinite(out[0]), fin)
    assert np.array_equal(bits(out[0])[fin], bits(u)[fin])
    ok = np.isfinite(want_tr)
    assert np.array_equal(bits(got_tr)[ok], bits(want_tr)[ok])


def test_diffusion_special_values_bitwise(sf, port):
    """Temporal blocking keeps subnormals and signed zeros (radius 1 and 4)."""
    from fractions import Fraction
    for order in (2, 8):
        n, nt = 133, 17
        rng = np.random.default_rng(900 + order)
        u = rng.standard_normal((2, n, n)).astype(np.float32)
        pick = rng.random((2, n, n))
        u[pick < 0.2] = -0.0
        u[(pick >= 0.2) & (pick < 0.5)] *= np.float32(1e-39)
        cfg = sf.DiffusionConfig(nx=n, ny=n, alpha=Fraction(1, 3), dx=Fraction(1, n - 1),
                                 dy=Fraction(1, n - 1), nt=nt, order=order)
        b = sf.make_diffusion_operator(cfg)
        b.u.data[...] = u
        b.op.apply()
        ref = u.copy()
        port.diffusion_run(ref, order, (1, 3), (1, n - 1), nt)
        assert np.array_equal(bits(b.u.data), bits(ref))


@pytest.mark.parametrize("order", [4, 8, 12])
@pytest.mark.parametrize("forward", [True, False])
def test_zero_eta_boxes_special_values(sf, port, order, forward):
    """All-zero eta boxes (skipped loads, 0.0f operands) with signed-zero,
    subnormal and infinite wavefield values and zero / negative-zero /
    subnormal m (infinite or huge t3): still the CPU oracle's bits wherever
    the result is finite, and the same non-finite pattern."""
    shape = (44, 53, 100)
    nt = 5
    c = random_case(port, shape, order, seed=700 + order + 2 * forward)
    rng = c["rng"]
    eta = np.zeros(shape, np.float32)          # almost every box is +0.0
    eta[:4] = c["eta"][:4]
    m = c["m"].copy()
    mp = rng.random(shape)
    m[mp < 0.02] = 0.0
    m[(mp >= 0.02) & (mp < 0.04)] = -0.0
    m[(mp >= 0.04) & (mp < 0.06)] = 1e-40
    m[(mp >= 0.06) & (mp < 0.08)] = 1e-30
    u0 = (1e-3 * rng.standard_normal((3,) + shape)).astype(np.float32)
    pick = rng.random((3,) + shape)
    u0[pick < 0.2] = 0.0
    u0[(pick >= 0.2) & (pick < 0.4)] = -0.0
    sub = (pick >= 0.4) & (pick < 0.5)
    u0[sub] = (rng.standard_normal(sub.sum()) * 1e-39).astype(np.float32)
    u0[1, 20, 26, 50] = np.inf                 # a few infinities (they spread R planes per step)
    u0[0, 30, 10, 80] = -np.inf
    u0[2, 12, 40, 20] = np.inf
    src = rng.standard_normal((nt, 3)).astype(np.float32)
    rec = rng.standard_normal((nt, 17)).astype(np.float32)
    s_in, r_in = (src, np.zeros_like(rec)) if forward else (np.zeros_like(src), rec)
    out = run_plan_raw(sf, shape, order, forward, c["dt"], 10.0, nt, m, eta, s_in.copy(),
                       c["src_ci"], c["src_w"], r_in.copy(), c["rec_ci"], c["rec_w"], u=u0.copy())
    coefs = port.coefs(3, order, forward, c["dt"], 10.0)
    u = u0.copy()
    if forward:
        port.acoustic_run(coefs, u, m, eta, s_in.copy(), c["src_ci"], c["src_w"], r_in.copy(),
                          c["rec_ci"], c["rec_w"], nt)
    else:
        port.acoustic_run(coefs, u, m, eta, r_in.copy(), c["rec_ci"], c["rec_w"], s_in.copy(),
                          c["src_ci"], c["src_w"], nt)
    fin = np.isfinite(u)
    assert np.array_equal(np.isfinite(out[0]), fin)
    assert np.array_equal(bits(out[0])[fin], bits(u)[fin])
    assert (~fin).any() and fin.sum() > 0.2 * fin.size


@pytest.mark.parametrize("order", [4, 8, 12, 16])
@pytest.mark.parametrize("forward", [True, False])
@pytest.mark.parametrize("knobs", [{}, {"SF_IO_STEPS": "1"}, {"SF_IO_STEPS": "3"},
                                   {"SF_IO_STEPS": "50"}, {"SF_IO_CHUNK_PLANES": "64"},
                                   {"SF_IO_STEPS": "4", "SF_IO_TAIL_STEPS": "0"},
                                   {"SF_IO_STEPS": "4", "SF_IO_TAIL_STEPS": "1"},
                                   {"SF_IO_STEPS": "4", "SF_IO_TAIL_STEPS": "2"},
                                   {"SF_IO_STEPS": "6", "SF_IO_TAIL_STEPS": "7",
                                    "SF_IO_CHUNK_PLANES": "64"},
                                   {"SF_NO_IO_OVERLAP": "1"}],
                         ids=lambda k: ",".join(f"{a}={b}" for a, b in k.items()) or "auto")
def test_invoke_overlapped_upload_bitwise(sf, port, monkeypatch, order, forward, knobs):
    """sf_acoustic_apply with the upload hidden behind the first time steps
    (plane chunks on a copy stream, the first K steps time-skewed behind the
    upload front, plan.cu invoke_overlapped) and the copy back hidden behind
    the last K2 steps (skewed so low planes become final first; with K = 1 or
    3 of the 19 steps the tail takes all the others): bitwise the oracle for
    every chunking, K and K2, with a random initial state in all three slots and point
    sets spread over every plane -- the boundary strips the stencil never
    writes, chunk seams, colliding cells -- so injection and sampling per plane
    range are exercised in both directions."""
    monkeypatch.setenv("SF_IO_OVERLAP", "1")  # small grids take the plain path by default
    for k, v in knobs.items():
        monkeypatch.setenv(k, v)
    r = order // 2
    shape = (131, 30, 70)  # five 32-plane chunks (the last one partial)
    nt = 19
    rng = np.random.default_rng(1000 + order + forward)
    v = 1500.0 + 3000.0 * rng.random(shape)
    m, eta = port.medium_from_velocity(v, 5, 10.0, 1500.0)
    dt = min(0.4 * 10.0 / 4500.0, port.stable_dt(3, order, 10.0, 4500.0, 4500.0))

    def pts(n):
        c = np.stack([rng.uniform(0.0, (e - 1.001) * 10.0, n) for e in shape], 1)
        # planes next to both faces, on chunk seams and in the middle
        z = np.concatenate([[0.2, 1.5, r - 0.5, r + 0.5, 30.7, 31.5, 32.2, 63.9, 95.5, 127.1,
                             shape[0] - r - 1.5, shape[0] - r - 0.5, shape[0] - 1.9],
                            rng.uniform(0.0, shape[0] - 1.001, max(0, n - 13))])[:n]
        c[:, 0] = z * 10.0
        return c
    src_c, rec_c = pts(21), pts(40)
    src_c[1] = src_c[0] + 0.1 * 10.0 * rng.random(3) * [0.0, 1.0, 1.0]  # shared cells
    src_ci, src_w = port.interp(src_c, 10.0, shape)
    rec_ci, rec_w = port.interp(rec_c, 10.0, shape)
    u0 = (1e-3 * rng.standard_normal((3,) + shape)).astype(np.float32)
    if forward:
        src = rng.standard_normal((nt, 21)).astype(np.float32)
        rec = np.zeros((nt, 40), np.float32)
    else:
        src = np.zeros((nt, 21), np.float32)
        rec = rng.standard_normal((nt, 40)).astype(np.float32)
    out = run_plan_raw(sf, shape, order, forward, dt, 10.0, nt, m, eta, src.copy(), src_ci, src_w,
                       rec.copy(), rec_ci, rec_w, u=u0.copy())
    coefs = port.coefs(3, order, forward, dt, 10.0)
    u = u0.copy()
    if forward:
        port.acoustic_run(coefs, u, m, eta, src, src_ci, src_w, rec, rec_ci, rec_w, nt)
        assert_parity(out[6], rec)
    else:
        port.acoustic_run(coefs, u, m, eta, rec, rec_ci, rec_w, src, src_ci, src_w, nt)
        assert_parity(out[3], src)
    assert_parity(out[0], u)
    assert np.abs(u).max() > 0

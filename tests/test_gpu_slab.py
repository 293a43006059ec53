"""Depth-slab decomposition on the GPU: an in-process chain of slab plans
(halo copies device to device, include/sf_b200.h sf_slab_chain_run) must be
bitwise the single-domain plan, forward and adjoint, with sources and
receivers straddling slab boundaries. One GPU runs all slabs; the multi-GPU
transport (NCCL send/recv, one process per GPU) reuses the same slab plans
and the same per-step order (stencil, owned injection, exchange, sampling).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a).view(np.uint32)


@pytest.mark.parametrize("order,forward,nslabs,shape", [
    (4, True, 3, (67, 40, 45)), (8, False, 2, (67, 40, 45)), (2, True, 4, (67, 40, 45)),
    (16, True, 2, (67, 40, 45)),
    # wide enough laterally for all-zero eta boxes (skipped loads) in every slab
    (4, True, 3, (67, 60, 140)), (8, False, 2, (58, 70, 140)), (12, True, 2, (58, 60, 140))])
def test_slab_chain_matches_single_domain(port, order, forward, nslabs, shape):
    import paper_1609_03361_b200 as sf
    from paper_1609_03361_b200.slab import SlabPartition, SlabRun, assemble, chain_run
    from test_gpu_parity import run_plan_raw
    nt = 20
    r = order // 2
    rng = np.random.default_rng(order)
    v = 1500.0 + 3000.0 * rng.random(shape)
    m, eta = port.medium_from_velocity(v, 5, 10.0, 1500.0)
    dt = min(0.4 * 10.0 / 4500.0, port.stable_dt(3, order, 10.0, 4500.0, 4500.0))
    bounds = [SlabPartition.split(shape[0], r, nslabs, g).own_begin for g in range(1, nslabs)]
    # points near every slab boundary plus random ones
    pts = []
    for b in bounds:
        for dz in (-1.3, -0.4, 0.2, 0.9):
            pts.append([(b + dz) * 10.0, rng.uniform(r + 1, shape[1] - 2 - r) * 10.0,
                        rng.uniform(r + 1, shape[2] - 2 - r) * 10.0])
    for _ in range(6):
        pts.append([rng.uniform(r + 1, shape[0] - 2 - r) * 10.0,
                    rng.uniform(r + 1, shape[1] - 2 - r) * 10.0,
                    rng.uniform(r + 1, shape[2] - 2 - r) * 10.0])
    pts = np.array(pts)
    src_c, rec_c = pts[::2], pts[1::2]
    src_ci, src_w = port.interp(src_c, 10.0, shape)
    rec_ci, rec_w = port.interp(rec_c, 10.0, shape)
    ns, nr = len(src_ci), len(rec_ci)
    if forward:
        src = rng.standard_normal((nt, ns)).astype(np.float32)
        rec = np.zeros((nt, nr), np.float32)
    else:
        src = np.zeros((nt, ns), np.float32)
        rec = rng.standard_normal((nt, nr)).astype(np.float32)
    ref = run_plan_raw(sf, shape, order, forward, dt, 10.0, nt, m, eta, src.copy(), src_ci, src_w,
                       rec.copy(), rec_ci, rec_w)
    slabs = [SlabRun(SlabPartition.split(shape[0], r, nslabs, g), shape, order, forward, nt, dt,
                     10.0, m, eta, src, src_ci, src_w, rec, rec_ci, rec_w) for g in range(nslabs)]
    chain_run(slabs, 0, nt)
    if shape[2] >= 140:  # the wide cases: every slab skipped some all-zero eta boxes
        import ctypes as C
        from paper_1609_03361_b200 import _lib
        for sl in slabs:
            frac = C.c_double()
            assert _lib.lib.sf_plan_eta_skip_fraction(sl.plan, C.byref(frac)) == 0
            assert frac.value > 0.0
    u, s_tr, r_tr = assemble(slabs, shape, nt, ns, nr)
    assert np.abs(ref[0]).max() > 0
    assert np.array_equal(bits(u), bits(ref[0]))
    if forward:
        assert np.array_equal(bits(r_tr), bits(ref[6]))
    else:
        assert np.array_equal(bits(s_tr), bits(ref[3]))
    for s in slabs:
        s.close()


def test_slab_desc_validation():
    import ctypes as C
    import paper_1609_03361_b200 as sf
    from paper_1609_03361_b200 import _lib
    d = _lib.AcousticDesc()
    d.ndim = 3
    d.shape[0], d.shape[1], d.shape[2] = 20, 16, 16
    d.space_order, d.forward, d.nt, d.dt, d.spacing, d.n_src, d.n_rec = 4, 1, 2, 1e-3, 10.0, 1, 1
    bad = _lib.SlabDesc(40, 0, 0, 19)  # shape[0] should be 21 (19 owned + 2 halo)
    plan = C.c_void_p()
    assert _lib.lib.sf_acoustic_plan_create_slab(C.byref(d), C.byref(bad), 0, C.byref(plan)) == \
        _lib.SF_ERR_INVALID
    ok = _lib.SlabDesc(40, 0, 0, 18)
    assert _lib.lib.sf_acoustic_plan_create_slab(C.byref(d), C.byref(ok), 0, C.byref(plan)) == 0
    _lib.lib.sf_plan_destroy(plan)
    del sf


def test_nccl_single_rank_plumbing(port):
    """The one-process-per-GPU transport on this box's single GPU: NCCL is
    dlopen'd (PyTorch's copy when loaded), a 1-rank communicator is created
    from sf_nccl_unique_id and attached to a whole-grid slab, and the run is
    bitwise the single-domain plan (no neighbour, so no exchange is issued)."""
    import torch  # noqa: F401  (brings PyTorch's NCCL into the process)
    import paper_1609_03361_b200 as sf
    from paper_1609_03361_b200.slab import SlabPartition, SlabRun, assemble, nccl_unique_id
    from test_gpu_parity import run_plan_raw
    shape, order, nt = (40, 36, 44), 8, 12
    r = order // 2
    rng = np.random.default_rng(3)
    v = 1500.0 + 3000.0 * rng.random(shape)
    m, eta = port.medium_from_velocity(v, 5, 10.0, 1500.0)
    dt = min(0.4 * 10.0 / 4500.0, port.stable_dt(3, order, 10.0, 4500.0, 4500.0))
    src_ci, src_w = port.interp(np.array([[200.0, 180.0, 210.0]]), 10.0, shape)
    rec_ci, rec_w = port.interp(np.array([[150.0, 100.0 + 9 * i, 120.0] for i in range(7)]),
                                10.0, shape)
    src = rng.standard_normal((nt, 1)).astype(np.float32)
    rec = np.zeros((nt, 7), np.float32)
    ref = run_plan_raw(sf, shape, order, True, dt, 10.0, nt, m, eta, src.copy(), src_ci, src_w,
                       rec.copy(), rec_ci, rec_w)
    slab = SlabRun(SlabPartition.split(shape[0], r, 1, 0), shape, order, True, nt, dt, 10.0, m,
                   eta, src, src_ci, src_w, rec, rec_ci, rec_w)
    slab.attach_nccl(nccl_unique_id(), 1, 0)
    slab.run(0, nt)
    u, _, r_tr = assemble([slab], shape, nt, 1, 7)
    assert np.array_equal(bits(u), bits(ref[0]))
    assert np.array_equal(bits(r_tr), bits(ref[6]))
    slab.close()

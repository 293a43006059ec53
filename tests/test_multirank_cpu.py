"""Multi-rank depth-slab path on CPU: world_size 2 over gloo.

Each rank owns a slab of the global grid as laid out by
paper_1609_03361_b200.slab.SlabPartition (the same bookkeeping the GPU
drivers use), advances it with the oracle's stencil (test-side stand-in for
the GPU kernel), applies its share of the injection and sampling in the
reference's fp32 order, and swaps r halo planes with its neighbour over gloo
after injection. The assembled result must be bitwise the single-domain run.
"""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT

SHAPE = (37, 22, 26)
ORDER = 4
NT = 12


def make_case():
    import sys
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_lib import Port
    port = Port()
    rng = np.random.default_rng(42)
    v = 1500.0 + 1000.0 * rng.random(SHAPE)
    m, eta = port.medium_from_velocity(v, 4, 10.0, 1500.0)
    dt = 0.4 * 10.0 / 2500.0
    # sources/receivers straddling the slab boundary (plane 18/19 for world 2)
    src_c = np.array([[17.6, 11.2, 12.3], [18.4, 8.1, 9.9], [5.5, 10.0, 10.0]]) * 10.0
    rec_c = np.array([[17.3 + 0.37 * i, 6.0 + 0.5 * i, 7.0 + 0.4 * i] for i in range(9)]) * 10.0
    src_ci, src_w = port.interp(src_c, 10.0, SHAPE)
    rec_ci, rec_w = port.interp(rec_c, 10.0, SHAPE)
    src = rng.standard_normal((NT, 3)).astype(np.float32)
    return port, m, eta, dt, src, src_ci, src_w, rec_ci, rec_w


def inject(u, m, row, ci, w, scale, own):
    """build_inject order: p ascending, corners in bit order; owned planes only."""
    s = np.float32(scale)
    for p in range(ci.shape[0]):
        for k in range(8):
            c = (ci[p, 0] + (k & 1), ci[p, 1] + ((k >> 1) & 1), ci[p, 2] + ((k >> 2) & 1))
            if not (own[0] <= c[0] < own[1]):
                continue
            d = np.float32(np.float32(np.float32(s * row[p]) * w[p, k]) / m[c])
            u[c] = np.float32(d + u[c])


def sample(u, ci, w):
    out = np.zeros(ci.shape[0], np.float32)
    for p in range(ci.shape[0]):
        acc = None
        for k in range(8):
            c = (ci[p, 0] + (k & 1), ci[p, 1] + ((k >> 1) & 1), ci[p, 2] + ((k >> 2) & 1))
            t = np.float32(w[p, k] * u[c])
            acc = t if acc is None else np.float32(acc + t)
        out[p] = acc
    return out


def stencil_step(port, coefs, out, cur, prev, m, eta):
    """One forward stencil sweep on a (local) array with the oracle: the port
    runs t = 0 with prev = slot 2, cur = slot 0, out = slot 1."""
    u3 = np.ascontiguousarray(np.stack([cur, out, prev]))
    z_ser = np.zeros((1, 1), np.float32)  # no sparse points: injection/sampling done by caller
    z_ci = np.zeros((0, 3), np.int32)
    z_w = np.zeros((0, 8), np.float32)
    port.acoustic_run(coefs, u3, m, eta, z_ser, z_ci, z_w, z_ser.copy(), z_ci, z_w, 1, 1)
    out[...] = u3[1]


def run_single(case):
    port, m, eta, dt, src, src_ci, src_w, rec_ci, rec_w = case
    c = port.coefs(3, ORDER, True, dt, 10.0)
    u = np.zeros((3,) + SHAPE, np.float32)
    rec = np.zeros((NT, rec_ci.shape[0]), np.float32)
    port.acoustic_run(c, u, m, eta, src.copy(), src_ci, src_w, rec, rec_ci, rec_w, NT, 1)
    return u, rec


def worker(rank, world, port_no, result_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_no)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, ROOT)
    from paper_1609_03361_b200.slab import SlabPartition
    case = make_case()
    port, m, eta, dt, src, src_ci, src_w, rec_ci, rec_w = case
    r = ORDER // 2
    part = SlabPartition.split(SHAPE[0], r, world, rank)
    sl = part.local()
    lm, leta = np.ascontiguousarray(m[sl]), np.ascontiguousarray(eta[sl])
    lshape = (part.local_n0,) + SHAPE[1:]
    u = [np.zeros(lshape, np.float32) for _ in range(3)]
    inj = np.nonzero(part.injecting(src_ci))[0]
    smp = np.nonzero(part.sampling(rec_ci))[0]
    l_src_ci = part.to_local(src_ci[inj])
    l_rec_ci = part.to_local(rec_ci[smp])
    own = (part.owned_local().start, part.owned_local().stop)
    coefs = port.coefs(3, ORDER, True, dt, 10.0)
    traces = np.zeros((NT, len(smp)), np.float32)
    for t in range(NT):
        prev, cur, out = u[(t + 2) % 3], u[t % 3], u[(t + 1) % 3]
        stencil_step(port, coefs, out, cur, prev, lm, leta)
        inject(out, lm, src[t, inj], l_src_ci, src_w[inj], coefs.src_scale, own)
        reqs = []
        bufs = {}
        if part.has_lower:
            reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(out[part.send_lower()])),
                                   rank - 1))
            bufs["lo"] = torch.zeros((r,) + SHAPE[1:])
            reqs.append(dist.irecv(bufs["lo"], rank - 1))
        if part.has_upper:
            reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(out[part.send_upper()])),
                                   rank + 1))
            bufs["hi"] = torch.zeros((r,) + SHAPE[1:])
            reqs.append(dist.irecv(bufs["hi"], rank + 1))
        for q in reqs:
            q.wait()
        if "lo" in bufs:
            out[part.recv_lower()] = bufs["lo"].numpy()
        if "hi" in bufs:
            out[part.recv_upper()] = bufs["hi"].numpy()
        traces[t] = sample(out, l_rec_ci, rec_w[smp])
    # gather owned planes and traces on rank 0
    payload = {"own": (part.own_begin, part.own_end),
               "u": np.stack([x[part.owned_local()] for x in u]), "smp": smp, "traces": traces}
    gathered = [None] * world
    dist.all_gather_object(gathered, payload)
    if rank == 0:
        g_u = np.zeros((3,) + SHAPE, np.float32)
        g_rec = np.zeros((NT, rec_ci.shape[0]), np.float32)
        seen = np.zeros(rec_ci.shape[0], int)
        for pl in gathered:
            b, e = pl["own"]
            g_u[:, b:e] = pl["u"]
            g_rec[:, pl["smp"]] = pl["traces"]
            seen[pl["smp"]] += 1
        np.savez(result_path, u=g_u, rec=g_rec, seen=seen)
    dist.barrier()
    dist.destroy_process_group()


def test_slab_partition_bookkeeping():
    from paper_1609_03361_b200.slab import SlabPartition
    for n0, r, world in [(37, 2, 2), (281 * 4, 4, 4), (100, 8, 8), (64, 1, 3)]:
        parts = [SlabPartition.split(n0, r, world, g) for g in range(world)]
        assert parts[0].own_begin == 0 and parts[-1].own_end == n0
        for a, b in zip(parts, parts[1:]):
            assert a.own_end == b.own_begin
            assert a.send_upper().stop - a.send_upper().start == r
            # what a sends up lands exactly in b's lower halo (global planes)
            assert (a.plane0 + a.send_upper().start == b.plane0 + b.recv_lower().start)
            assert (b.plane0 + b.send_lower().start == a.plane0 + a.recv_upper().start)
        for p in parts:
            assert p.local_n0 == (p.own_end - p.own_begin) + r * p.has_lower + r * p.has_upper
    with pytest.raises(ValueError):
        SlabPartition.split(10, 4, 4, 0)
    # every receiver has exactly one sampling owner; injection owners cover corners
    rng = np.random.default_rng(0)
    ci = np.stack([rng.integers(0, 98, 500), rng.integers(0, 10, 500), rng.integers(0, 10, 500)], 1)
    parts = [SlabPartition.split(100, 2, 4, g) for g in range(4)]
    owners = sum(p.sampling(ci).astype(int) for p in parts)
    assert np.all(owners == 1)
    for p in parts:
        loc = p.to_local(ci[p.injecting(ci)])
        assert loc[:, 0].min() >= 0 and loc[:, 0].max() + 1 < p.local_n0


def test_two_rank_gloo_slabs_match_single_domain(tmp_path):
    case = make_case()
    u_ref, rec_ref = run_single(case)
    path = str(tmp_path / "res.npz")
    port_no = 29500 + (os.getpid() % 1000)
    mp.spawn(worker, args=(2, port_no, path), nprocs=2, join=True)
    res = np.load(path)
    assert np.all(res["seen"] == 1)
    assert np.abs(u_ref).max() > 0
    assert np.array_equal(res["u"].view(np.uint32), u_ref.view(np.uint32))
    assert np.array_equal(res["rec"].view(np.uint32), rec_ref.view(np.uint32))

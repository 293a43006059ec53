"""Depth-slab decomposition of the acoustic grid across GPUs.

The reference has no domain decomposition; this is the
B200 build's multi-GPU path. The grid is split along storage axis 0 (depth,
the slowest axis), so every message is a run of contiguous planes. Rank g
owns global planes [own_begin, own_end) and stores r = space_order/2 halo
planes on each internal side. Per time step (include/sf_b200.h, slab plans):

  1. stencil on owned interior planes,
  2. injection into the corners the slab owns (contributions to other
     slabs' corners are applied by those slabs, in the same p order),
  3. halo exchange of the level just written (after injection, so halos
     carry injected values): first r owned planes down, last r up,
  4. sampling by the slab that owns each receiver's lower corner plane
     (its upper corner may sit in the halo, which is now current).

Every owned value is computed with the identical arithmetic as the single
domain run, so the decomposition is bitwise transparent. This module is the
host-side bookkeeping shared by the GPU drivers (in-process chain, or one
process per GPU over NCCL) and by the CPU gloo tests.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class SlabPartition:
    global_n0: int
    r: int
    world: int
    rank: int
    own_begin: int
    own_end: int

    @classmethod
    def split(cls, global_n0: int, r: int, world: int, rank: int) -> "SlabPartition":
        """Balanced contiguous split; the first global_n0 % world ranks get one
        extra plane. Every slab must own at least r planes."""
        base, extra = divmod(global_n0, world)
        begin = rank * base + min(rank, extra)
        end = begin + base + (1 if rank < extra else 0)
        if end - begin < r:
            raise ValueError(f"slab of rank {rank} owns {end - begin} planes < r = {r}")
        return cls(global_n0, r, world, rank, begin, end)

    @property
    def plane0(self) -> int:
        return max(self.own_begin - self.r, 0)

    @property
    def plane_end(self) -> int:
        return min(self.own_end + self.r, self.global_n0)

    @property
    def local_n0(self) -> int:
        return self.plane_end - self.plane0

    @property
    def has_lower(self) -> bool:
        return self.own_begin > 0

    @property
    def has_upper(self) -> bool:
        return self.own_end < self.global_n0

    def local(self) -> slice:
        """Global planes stored by this slab (owned + halos)."""
        return slice(self.plane0, self.plane_end)

    def owned_local(self) -> slice:
        return slice(self.own_begin - self.plane0, self.own_end - self.plane0)

    # halo exchange ranges, local plane indices
    def send_lower(self) -> slice:
        lo = self.own_begin - self.plane0
        return slice(lo, lo + self.r)

    def recv_lower(self) -> slice:
        lo = self.own_begin - self.plane0
        return slice(lo - self.r, lo)

    def send_upper(self) -> slice:
        hi = self.own_end - self.plane0
        return slice(hi - self.r, hi)

    def recv_upper(self) -> slice:
        hi = self.own_end - self.plane0
        return slice(hi, hi + self.r)

    # sparse points (global cell indices ci[p][0] on axis 0)
    def injecting(self, ci: np.ndarray) -> np.ndarray:
        """Points with at least one corner plane (ci0 or ci0+1) owned."""
        c0 = ci[:, 0]
        return (c0 + 1 >= self.own_begin) & (c0 < self.own_end)

    def sampling(self, ci: np.ndarray) -> np.ndarray:
        """Points whose lower corner plane is owned (one owner per point)."""
        c0 = ci[:, 0]
        return (c0 >= self.own_begin) & (c0 < self.own_end)

    def to_local(self, ci: np.ndarray) -> np.ndarray:
        out = np.array(ci, dtype=np.int32, copy=True)
        out[:, 0] -= self.plane0
        return out

    def slab_desc(self):
        from ._lib import SlabDesc
        return SlabDesc(self.global_n0, self.plane0, self.own_begin, self.own_end)


class SlabRun:
    """One slab of an acoustic run: a slab plan plus its local buffers.

    `field` (3 slots), m, eta are the global arrays (only this slab's planes
    are read; with local_medium=True m / eta hold just the local planes); src/rec series, cell indices and weights are global too and
    are filtered/translated here.
    """

    def __init__(self, part: SlabPartition, shape, space_order, forward, nt, dt, spacing, m, eta,
                 src, src_ci, src_w, rec, rec_ci, rec_w, u=None, device=0,
                 local_medium=False):
        from . import _lib
        from .api import check
        self.part = part
        self.forward = forward
        sl = part.local()
        lshape = (part.local_n0,) + tuple(shape[1:])
        inj_ci, smp_ci = (src_ci, rec_ci) if forward else (rec_ci, src_ci)
        self.inj_mask = part.injecting(inj_ci)
        self.smp_mask = part.sampling(smp_ci)
        # every plan needs non-empty point sets: keep one zero-weight dummy
        # sampled at the first local cell when a set is empty (its trace is
        # never read back)

        def subset(series, ci, w, mask):
            idx = np.nonzero(mask)[0]
            if len(idx) == 0:
                return (np.zeros((nt, 1), np.float32), np.zeros((1, 3), np.int32),
                        np.zeros((1, 8), np.float32), idx)
            return (np.ascontiguousarray(series[:, idx], np.float32), part.to_local(ci[idx]),
                    np.ascontiguousarray(w[idx], np.float32), idx)

        if forward:
            s_ser, s_ci, s_w, self.src_idx = subset(src, src_ci, src_w, self.inj_mask)
            r_ser, r_ci, r_w, self.rec_idx = subset(rec, rec_ci, rec_w, self.smp_mask)
        else:
            r_ser, r_ci, r_w, self.rec_idx = subset(rec, rec_ci, rec_w, self.inj_mask)
            s_ser, s_ci, s_w, self.src_idx = subset(src, src_ci, src_w, self.smp_mask)
        # a dummy point set must not inject anything
        if forward and len(self.src_idx) == 0:
            s_ser[:] = 0
        if not forward and len(self.rec_idx) == 0:
            r_ser[:] = 0
        d = _lib.AcousticDesc()
        d.ndim = 3
        for i, e in enumerate(lshape):
            d.shape[i] = e
        d.space_order, d.forward, d.nt, d.dt, d.spacing = space_order, int(forward), nt, dt, spacing
        d.n_src, d.n_rec = s_ci.shape[0], r_ci.shape[0]
        plan = C.c_void_p()
        check(_lib.lib.sf_acoustic_plan_create_slab(C.byref(d), C.byref(part.slab_desc()), device,
                                                    C.byref(plan)))
        self.plan = plan
        u_loc = (np.zeros((3,) + lshape, np.float32) if u is None
                 else np.ascontiguousarray(u[:, sl], np.float32))
        if local_medium:  # m / eta already hold just this slab's planes
            if m.shape[0] != part.local_n0 or eta.shape[0] != part.local_n0:
                raise ValueError("local medium must hold the slab's local planes")
            m_loc, eta_loc = m, eta
        else:
            m_loc, eta_loc = m[sl], eta[sl]
        self.bufs = [u_loc, np.ascontiguousarray(m_loc, np.float32),
                     np.ascontiguousarray(eta_loc, np.float32), s_ser, s_ci, s_w, r_ser, r_ci,
                     r_w]
        argv = (C.c_void_p * 9)(*[b.ctypes.data for b in self.bufs])
        check(_lib.lib.sf_plan_upload(self.plan, argv, 9))

    def download(self):
        from . import _lib
        from .api import check
        argv = (C.c_void_p * 9)(*[b.ctypes.data for b in self.bufs])
        check(_lib.lib.sf_plan_download(self.plan, argv, 9))
        return self.bufs

    def attach_nccl(self, uid: bytes, world: int, rank: int):
        from . import _lib
        from .api import check
        check(_lib.lib.sf_plan_attach_nccl(self.plan, uid, world, rank))

    def run(self, b, e):
        from . import _lib
        from .api import check
        check(_lib.lib.sf_plan_run(self.plan, b, e))
        check(_lib.lib.sf_plan_synchronize(self.plan))

    def close(self):
        from . import _lib
        if self.plan:
            _lib.lib.sf_plan_destroy(self.plan)
            self.plan = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def chain_run(slabs: list[SlabRun], b: int, e: int):
    """Steps [b, e) of adjacent slabs in this process (halo copies D2D)."""
    from . import _lib
    from .api import check
    arr = (C.c_void_p * len(slabs))(*[s.plan.value for s in slabs])
    check(_lib.lib.sf_slab_chain_run(arr, len(slabs), b, e))


def assemble(slabs: list[SlabRun], shape, nt, n_src, n_rec):
    """Global field slots and traces from downloaded slabs."""
    u = np.zeros((3,) + tuple(shape), np.float32)
    src = np.zeros((nt, n_src), np.float32)
    rec = np.zeros((nt, n_rec), np.float32)
    for s in slabs:
        bufs = s.download()
        p = s.part
        u[:, p.own_begin:p.own_end] = bufs[0][:, p.owned_local()]
        if s.forward:
            rec[:, s.rec_idx] = bufs[6][:, :len(s.rec_idx)]
        else:
            src[:, s.src_idx] = bufs[3][:, :len(s.src_idx)]
    return u, src, rec


def nccl_unique_id() -> bytes:
    from . import _lib
    from .api import check
    buf = C.create_string_buffer(128)
    check(_lib.lib.sf_nccl_unique_id(buf, 128))
    return buf.raw

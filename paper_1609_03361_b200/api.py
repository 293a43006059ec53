"""Host-side mirror of the reference's public API for the hot path.

Names, argument meaning and error behaviour follow stencilforge
(/root/reference/proj/include/sf/*.hpp) so code and tests written against
the reference read the same here:

  sf::AcousticModel / acoustic_build / acoustic_forward / acoustic_adjoint /
  adjoint_test / adjoint_test_with          acoustic.hpp:17-91
  sf::DiffusionConfig / diffusion_run       diffusion.hpp:13-51
  sf::Grid / GridFunction                   grid.hpp:32-139
  sf::SparsePointSet / interpolation_weights sparse.hpp:11-47
  sf::Operator::build / apply               op.hpp:37-84

Every buffer lives in host memory in the reference's dense layout; the
Operator's apply() hands them to the CUDA plan (include/sf_b200.h), which
keeps padded mirrors in HBM, runs all nt steps as a CUDA graph and copies the
results back. The folded constants, the injection CSR, the graph and the
memory layout are all built natively (csrc/); this module only arranges
buffers.
"""
from __future__ import annotations

import ctypes as C
import math
import re
from dataclasses import dataclass, field
from fractions import Fraction

import numpy as np

from . import _lib
from ._lib import lib


# ---------------------------------------------------------------------------
# errors (error.hpp:9-57)

class SfError(RuntimeError):
    pass


class InvalidShapeError(SfError):
    pass


class InvalidOrderError(SfError):
    pass


class CflViolationError(SfError):
    pass


class OutOfDomainError(SfError):
    pass


class SignatureMismatchError(SfError):
    pass


class KernelFailedError(SfError):
    pass


class CudaError(SfError):
    pass


_ERRORS = {
    _lib.SF_ERR_INVALID: InvalidShapeError,
    _lib.SF_ERR_CFL: CflViolationError,
    _lib.SF_ERR_OUT_OF_DOMAIN: OutOfDomainError,
    _lib.SF_ERR_SIGNATURE: SignatureMismatchError,
    _lib.SF_ERR_KERNEL: KernelFailedError,
    _lib.SF_ERR_CUDA: CudaError,
    _lib.SF_ERR_OOM: CudaError,
}


def check(rc: int):
    if rc != _lib.SF_OK:
        raise _ERRORS.get(rc, SfError)(_lib.last_error())


# ---------------------------------------------------------------------------
# grid data (grid.hpp:32-139)

def pinned_array(shape, dtype=np.float32, like=None):
    """Page-locked host array (numpy view of a pinned torch tensor; torch is
    plumbing only): async H2D / D2H copies run at the PCIe rate from these."""
    import torch
    tdt = {np.float32: torch.float32, np.int32: torch.int32}[np.dtype(dtype).type]
    t = torch.zeros(tuple(shape), dtype=tdt, pin_memory=True)
    a = t.numpy()  # shares (and keeps alive) the tensor's page-locked storage
    if like is not None:
        a[...] = like
    return a


class GridFunction:
    """Named buffer in the reference's dense layout (slot slowest)."""

    def __init__(self, name, shape, dtype=np.float32, time_order=None, space_order=2,
                 pinned=False):
        self.name = name
        self.time_order = time_order
        self.space_order = space_order
        if pinned:
            import torch  # plumbing only: page-locked host memory for fast H2D/D2H
            tdt = {np.float32: torch.float32, np.int32: torch.int32}[np.dtype(dtype).type]
            self._pin = torch.zeros(tuple(shape), dtype=tdt, pin_memory=True)
            self.data = self._pin.numpy()
        else:
            self.data = np.zeros(shape, dtype)

    @property
    def shape(self):
        return self.data.shape

    def slots(self):
        return self.time_order + 1 if self.time_order is not None else 1

    def space_shape(self):
        return self.data.shape[1:] if self.time_order is not None else self.data.shape

    def get(self, idx):
        return float(self.data[tuple(idx)])

    def set(self, idx, value):
        self.data[tuple(idx)] = value

    def view(self):
        return self.data.reshape(-1)

    def bytes(self):
        return self.data.nbytes

    def zero(self):
        self.data[...] = 0


class Grid:
    """Registry of GridFunctions; declaration order fixes argument order."""

    def __init__(self, pinned=False):
        self.functions: dict[str, GridFunction] = {}
        self.pinned = pinned

    def _insert(self, gf):
        if gf.name in self.functions:
            raise SfError(f"name already registered: {gf.name}")
        self.functions[gf.name] = gf
        return gf

    def create_dense(self, name, space_shape, space_order=2):
        _validate_shape_order(space_shape, space_order)
        return self._insert(GridFunction(name, tuple(space_shape), np.float32, None, space_order,
                                         self.pinned))

    def create_time(self, name, space_shape, time_order, space_order=2):
        _validate_shape_order(space_shape, space_order)
        if time_order < 1:
            raise InvalidOrderError(f"time_order must be >= 1, got {time_order}")
        return self._insert(GridFunction(name, (time_order + 1,) + tuple(space_shape),
                                         np.float32, time_order, space_order, self.pinned))

    def create_array(self, name, shape, dtype=np.float32):
        if any(e < 1 for e in shape):
            raise InvalidShapeError("array extent must be positive")
        return self._insert(GridFunction(name, tuple(shape), dtype, None, 0, self.pinned))

    def find(self, name):
        return self.functions.get(name)


def _validate_shape_order(shape, order):
    if len(shape) < 1 or len(shape) > 3:
        raise InvalidShapeError("expected 1-3 spatial dimensions")
    if order < 2 or order % 2:
        raise InvalidOrderError(f"space_order must be even and >= 2, got {order}")
    for e in shape:
        if e < order + 1:
            raise InvalidShapeError(f"extent {e} too small for order {order}")


# ---------------------------------------------------------------------------
# sparse points (sparse.hpp:11-47)

def interpolation_weights(coord, spacing, extents):
    """Enclosing cell and 2^d multilinear weights (f32) of one point."""
    coord = np.ascontiguousarray(coord, np.float64)
    ext = np.ascontiguousarray(extents, np.int64)
    nd = len(coord)
    cell = np.zeros(nd, np.int32)
    w = np.zeros(1 << nd, np.float32)
    rc = lib.sf_interpolation_weights(nd, coord, float(spacing), ext, cell, w)
    if rc == _lib.SF_ERR_OUT_OF_DOMAIN:
        raise OutOfDomainError("coordinate outside the grid")
    check(rc)
    return cell, w


class SparsePointSet:
    """Per-point series plus enclosing-cell indices and corner weights,
    registered as <name>, <name>_ci and <name>_w (sparse.cpp:43-75)."""

    def __init__(self, grid: Grid, name, coords, nt, spacing, field: GridFunction):
        if len(coords) == 0:
            raise OutOfDomainError("point set is empty")
        extents = field.space_shape()
        self.sdim = len(extents)
        self.np = len(coords)
        self.nt = nt
        self.data = grid.create_array(name, (nt, self.np), np.float32)
        self.ci = grid.create_array(name + "_ci", (self.np, self.sdim), np.int32)
        self.w = grid.create_array(name + "_w", (self.np, 1 << self.sdim), np.float32)
        for p, c in enumerate(coords):
            if len(c) != self.sdim:
                raise OutOfDomainError(f"point {p} has wrong rank")
            cell, w = interpolation_weights(c, spacing, extents)
            self.ci.data[p] = cell
            self.w.data[p] = w

    def num_points(self):
        return self.np

    def set_series(self, t, p, v):
        self.data.data[t, p] = v

    def series(self, t, p):
        return float(self.data.data[t, p])


# ---------------------------------------------------------------------------
# operators: a CUDA plan plus the grid buffers it binds (op.hpp:37-84)

class Operator:
    def __init__(self, plan_ptr, args: list[GridFunction]):
        self._plan = C.c_void_p(plan_ptr)
        self.args = args
        n = lib.sf_plan_num_args(self._plan)
        names = [lib.sf_plan_arg_name(self._plan, i).decode() for i in range(n)]
        if names != [a.name for a in args]:
            raise SignatureMismatchError(f"plan expects {names}")

    def __del__(self):
        try:
            if self._plan:
                lib.sf_plan_destroy(self._plan)
                self._plan = None
        except Exception:
            pass

    def signature(self):
        n = lib.sf_plan_num_args(self._plan)
        return [(lib.sf_plan_arg_name(self._plan, i).decode(),
                 lib.sf_plan_arg_bytes(self._plan, i)) for i in range(n)]

    def _argv(self, buffers=None):
        bufs = self.args if buffers is None else buffers
        if len(bufs) != len(self.args):
            raise SignatureMismatchError(f"expected {len(self.args)} buffers, got {len(bufs)}")
        for i, (b, want) in enumerate(zip(bufs, self.args)):
            if b is None or b.name != want.name:
                raise SignatureMismatchError(f"argument {i} must be {want.name}")
            if b.data.nbytes != lib.sf_plan_arg_bytes(self._plan, i):
                raise SignatureMismatchError(f"shape mismatch for {want.name}")
        arr = (C.c_void_p * len(bufs))(*[b.data.ctypes.data for b in bufs])
        return arr, len(bufs)

    def build(self):
        return self

    def apply(self, buffers=None):
        """All nt steps on the GPU; buffers updated in place. Returns 0."""
        argv, n = self._argv(buffers)
        check(lib.sf_plan_invoke(self._plan, argv, n))
        return 0

    # HBM-resident control (bench.py, multi-step drivers)
    def upload(self, buffers=None):
        argv, n = self._argv(buffers)
        check(lib.sf_plan_upload(self._plan, argv, n))

    def run(self, step_begin, step_end):
        check(lib.sf_plan_run(self._plan, step_begin, step_end))

    def synchronize(self):
        check(lib.sf_plan_synchronize(self._plan))

    def download(self, buffers=None):
        argv, n = self._argv(buffers)
        check(lib.sf_plan_download(self._plan, argv, n))

    def save_buffer(self, name, path):
        """save_buffer (grid.cpp:215-234) straight from the HBM mirror."""
        check(lib.sf_plan_save_buffer(self._plan, name.encode(), str(path).encode()))

    def load_buffer(self, name, path):
        """load_buffer (grid.cpp:236-254) straight into the HBM mirror."""
        check(lib.sf_plan_load_buffer(self._plan, name.encode(), str(path).encode()))

    def dump_csv(self, name, path, slot=0):
        """dump_csv (grid.cpp:256-273) of a 2D grid function from HBM."""
        check(lib.sf_plan_dump_csv(self._plan, name.encode(), str(path).encode(), slot))

    def save_series_text(self, name, path):
        """save_series_text (sparse.cpp:215-227) of "src"/"rec" from HBM."""
        check(lib.sf_plan_save_series_text(self._plan, name.encode(), str(path).encode()))

    KINDS = {0: "per-thread-load", 1: "tma", 2: "vector-tma", 3: "queue-vector-tma"}

    def autotune(self, tune_nt=5, repeats=3):
        """Operator::autotune (op.cpp:169-221) on the GPU: time every stencil
        variant on `tune_nt` steps of the uploaded state (restored before each
        run), keep the fastest. Returns [(description, median_seconds)], best."""
        ents = (_lib.TuneEntry * 64)()
        n = C.c_int()
        check(lib.sf_plan_autotune(self._plan, tune_nt, repeats, ents, 64, C.byref(n)))
        rep = []
        for e in ents[: min(n.value, 64)]:
            desc = (f"{self.KINDS[e.kind]} nx={e.tile_nx} ty={e.tile_ty} warps={e.vec_warps} "
                    f"stages={e.stages}")
            if e.kind == 2:  # vector ring: rows of four points per lane
                desc += f" rows/lane={max(1, e.tile_ty * e.tile_nx // (4 * e.vec_warps))}"
            rep.append((desc, e.median_ms / 1e3))
        best = min(rep, key=lambda x: x[1]) if rep else None
        return rep, best

    def eta_skip_fraction(self):
        """Fraction of interior point updates per step whose eta box the
        vector kernels skip (all +0.0); measurement hook for the roofline."""
        f = C.c_double()
        check(lib.sf_plan_eta_skip_fraction(self._plan, C.byref(f)))
        return f.value

    def time(self, stencil=True):
        """(total_ms, stencil_ms, kernel_launches) of one device-timed run."""
        tot = C.c_float()
        st = C.c_float()
        nl = C.c_int64()
        check(lib.sf_plan_time(self._plan, C.byref(tot), C.byref(st) if stencil else None,
                               C.byref(nl)))
        return tot.value, (st.value if stencil else None), nl.value


# ---------------------------------------------------------------------------
# acoustic application (acoustic.hpp:17-91)

_NUM = re.compile(r"[+-]?(?:\d+\.?\d*|\.\d+)(?:[eE][+-]?\d+)?")


def load_series_column(path) -> np.ndarray:
    """load_series_column (sparse.cpp:205-213): whitespace-separated numbers
    read with `in >> double` until the first token that does not parse (a
    numeric prefix is still taken, as the stream extraction does)."""
    try:
        with open(path) as f:
            text = f.read()
    except OSError as e:
        raise SfError(f"cannot open series file: {path}") from e
    out = []
    for tok in text.split():
        m = _NUM.match(tok)
        if not m:
            break
        out.append(float(m.group(0)))
        if m.end() != len(tok):
            break
    return np.asarray(out, np.float64)


def ricker_wavelet(f0, t, t0):
    return lib.sf_ricker(f0, t, t0)


def _stable_dt(ndim, order, spacing, v_top, v_bottom):
    v = lib.sf_stable_dt(ndim, order, spacing, v_top, v_bottom)
    if v < 0:
        raise InvalidOrderError(_lib.last_error())
    return v


@dataclass
class AcousticModel:
    shape: tuple = (60, 60)
    boundary_width: int = 10
    spacing: float = 15.0
    nt: int = 300
    dt: float = 0.0
    space_order: int = 2
    f0: float = 10.0
    v_top: float = 1500.0
    v_bottom: float = 2500.0
    src_coords: list = field(default_factory=list)
    rec_coords: list = field(default_factory=list)

    def dims(self):
        return len(self.shape)

    def stable_dt(self):
        return _stable_dt(self.dims(), self.space_order, self.spacing, self.v_top, self.v_bottom)

    def effective_dt(self):
        return self.dt if self.dt > 0 else self.stable_dt()

    def default_src(self):
        return [[(e / 2.0 + 0.31) * self.spacing for e in self.shape]]

    def default_rec(self, n=8):
        bw = self.boundary_width
        depth = (bw + 3 + (self.shape[0] - 2 * bw) / 4.0) * self.spacing
        lo = (bw + 2) * self.spacing
        hi = (self.shape[1] - bw - 3) * self.spacing
        out = []
        for i in range(n):
            c = [depth, lo + (hi - lo) * (i + 0.17) / n]
            while len(c) < len(self.shape):
                c.append((self.shape[len(c)] / 2.0 + 0.23) * self.spacing)
            out.append(c)
        return out


@dataclass
class AcousticSetup:
    grid: Grid
    field: GridFunction
    m: GridFunction
    eta: GridFunction
    src: SparsePointSet
    rec: SparsePointSet
    op: Operator
    nt: int
    dt: float


def build_medium(grid: Grid, model: AcousticModel, v_field=None, v_min=None, smooth=None,
                 device=0):
    """m and eta (acoustic.cpp:67-105); v_field overrides the two layers,
    `smooth` (a SmoothMedium of the model's shape) generates them on the GPU."""
    m = grid.create_dense("m", model.shape, model.space_order)
    eta = grid.create_dense("eta", model.shape, model.space_order)
    if smooth is not None:
        if tuple(smooth.shape) != tuple(model.shape):
            raise InvalidShapeError("smooth medium shape differs from the model")
        lo, hi = smooth.extrema(device=device)
        smooth.generate(lo, hi, device=device, out=(m.data, eta.data))
        return m, eta
    shape = np.asarray(model.shape, np.int64)
    vptr = None
    if v_field is not None:
        v_field = np.ascontiguousarray(v_field, np.float64)
        assert v_field.shape == tuple(model.shape)
        vptr = v_field.ctypes.data
    check(lib.sf_build_medium(len(model.shape), shape, model.boundary_width, model.spacing,
                              model.v_top, model.v_bottom, vptr,
                              float(v_min if v_min is not None else 0.0),
                              m.data.reshape(-1), eta.data.reshape(-1)))
    return m, eta


@dataclass
class SmoothMedium:
    """Seeded smooth random medium (configs C3/C4/C5): Gaussian-
    filtered hash noise rescaled to [v_lo, v_hi], then build_medium's m / eta
    (acoustic.cpp:67-105). Generated on the GPU from global indices
    (csrc/medium.cu), so a depth slab makes only its own planes; the global
    extrema come from `extrema()` over every slab (min / max over ranks)."""
    shape: tuple
    seed: int = 1234
    sigma: float = 8.0
    v_lo: float = 1500.0
    v_hi: float = 4500.0
    boundary_width: int = 40
    spacing: float = 10.0
    v_min: float = 1500.0

    def desc(self, a0_begin=0, a0_end=None):
        d = _lib.SmoothMediumDesc()
        for i, e in enumerate(self.shape):
            d.shape[i] = e
        d.a0_begin = a0_begin
        d.a0_end = self.shape[0] if a0_end is None else a0_end
        d.seed, d.sigma, d.v_lo, d.v_hi = self.seed, self.sigma, self.v_lo, self.v_hi
        d.boundary_width, d.spacing, d.v_min = self.boundary_width, self.spacing, self.v_min
        return d

    def extrema(self, a0_begin=0, a0_end=None, device=0):
        lo, hi = C.c_double(), C.c_double()
        check(lib.sf_smooth_extrema(C.byref(self.desc(a0_begin, a0_end)), device, C.byref(lo),
                                    C.byref(hi)))
        return lo.value, hi.value

    def generate(self, lo, hi, a0_begin=0, a0_end=None, device=0, out=None):
        """m, eta of global planes [a0_begin, a0_end) as dense host arrays."""
        e = self.shape[0] if a0_end is None else a0_end
        shp = (e - a0_begin,) + tuple(self.shape[1:])
        m, eta = out if out is not None else (np.empty(shp, np.float32), np.empty(shp, np.float32))
        assert m.shape == shp and eta.shape == shp and m.flags.c_contiguous
        check(lib.sf_smooth_medium(C.byref(self.desc(a0_begin, e)), lo, hi, device,
                                   m.ctypes.data, eta.ctypes.data))
        return m, eta

    def set_plan(self, op: "Operator", lo, hi):
        """Write m / eta straight into a plan's HBM mirrors (its own planes)."""
        check(lib.sf_plan_set_smooth_medium(op._plan, C.byref(self.desc()), lo, hi))


def _fill_series(pts: SparsePointSet, series, model: AcousticModel):
    nt, np_ = pts.nt, pts.np
    if series is not None and len(series):
        s = np.asarray(series, np.float64)
        if s.size != nt * np_:
            raise InvalidShapeError("series must be nt x num_points")
        pts.data.data[...] = s.reshape(nt, np_).astype(np.float32)
        return
    dt = model.effective_dt()
    t0 = 1.0 / model.f0
    vals = np.array([ricker_wavelet(model.f0, t * dt, t0) for t in range(nt)], np.float64)
    pts.data.data[...] = vals.astype(np.float32)[:, None]


def acoustic_build(model: AcousticModel, forward_run: bool, src_series=None, rec_series=None,
                   device=0, v_field=None, v_min=None, pinned=False,
                   smooth=None) -> AcousticSetup:
    """Configure without executing (acoustic.cpp:128-206)."""
    if model.dims() < 2 or model.dims() > 3:
        raise InvalidShapeError("acoustic model needs 2 or 3 dimensions")
    dt_s = model.effective_dt()
    if dt_s > model.stable_dt() * (1.0 + 1e-12):
        raise CflViolationError(f"dt {dt_s:f} exceeds stability bound {model.stable_dt():f}")
    grid = Grid(pinned=pinned)
    fname = "u" if forward_run else "v"
    fld = grid.create_time(fname, model.shape, 2, model.space_order)
    m, eta = build_medium(grid, model, v_field, v_min, smooth, device)
    src_coords = model.src_coords or model.default_src()
    rec_coords = model.rec_coords or model.default_rec()
    src = SparsePointSet(grid, "src", src_coords, model.nt, model.spacing, fld)
    rec = SparsePointSet(grid, "rec", rec_coords, model.nt, model.spacing, fld)
    if forward_run:
        _fill_series(src, src_series, model)
    else:
        _fill_series(rec, rec_series, model)
    desc = _lib.AcousticDesc()
    desc.ndim = model.dims()
    for i, e in enumerate(model.shape):
        desc.shape[i] = e
    desc.space_order = model.space_order
    desc.forward = int(forward_run)
    desc.nt = model.nt
    desc.dt = dt_s
    desc.spacing = model.spacing
    desc.n_src = src.np
    desc.n_rec = rec.np
    plan = C.c_void_p()
    check(lib.sf_acoustic_plan_create(C.byref(desc), device, C.byref(plan)))
    args = [fld, m, eta, src.data, src.ci, src.w, rec.data, rec.ci, rec.w]
    op = Operator(plan.value, args)
    return AcousticSetup(grid, fld, m, eta, src, rec, op, model.nt, dt_s)


def acoustic_forward(model: AcousticModel, src_series=None, **kw) -> AcousticSetup:
    s = acoustic_build(model, True, src_series=src_series, **kw)
    s.op.apply()
    return s


def acoustic_adjoint(model: AcousticModel, rec_residual, **kw) -> AcousticSetup:
    s = acoustic_build(model, False, rec_series=rec_residual, **kw)
    s.op.apply()
    return s


def _mt19937_64_uniform(seed, n, lo, hi):
    """std::mt19937_64(seed) + std::uniform_real_distribution<double>(lo, hi)
    as libstdc++ evaluates it (acoustic.cpp:230-235 draws x then y)."""
    mask = (1 << 64) - 1
    mt = [0] * 312
    mt[0] = seed & mask
    for i in range(1, 312):
        mt[i] = (6364136223846793005 * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i) & mask
    idx = 312
    out = np.empty(n, np.float64)
    for j in range(n):
        if idx >= 312:
            for i in range(312):
                x = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % 312] & 0x7FFFFFFF)
                xa = x >> 1
                if x & 1:
                    xa ^= 0xB5026F5AA96619E9
                mt[i] = mt[(i + 156) % 312] ^ xa
            idx = 0
        y = mt[idx]
        idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        c = float(y & mask) / 18446744073709551616.0
        if c >= 1.0:
            c = math.nextafter(1.0, 0.0)
        out[j] = c * (hi - lo) + lo
    return out


@dataclass
class AdjointTestResult:
    forward_product: float
    adjoint_product: float
    difference: float
    ratio: float
    degenerate: bool


def adjoint_test_with(model: AcousticModel, x, y, **kw) -> AdjointTestResult:
    """<Ax, y> vs <x, A^T y> (acoustic.cpp:239-270)."""
    fwd = acoustic_forward(model, x, **kw)
    nt = model.nt
    yv = np.asarray(y, np.float64).reshape(nt, -1)
    xv = np.asarray(x, np.float64).reshape(nt, -1)
    axy = 0.0
    recs = fwd.rec.data.data.astype(np.float64)
    for t in range(nt):
        for r in range(yv.shape[1]):
            axy += recs[t, r] * yv[t, r]
    adj = acoustic_adjoint(model, y, **kw)
    srcs = adj.src.data.data.astype(np.float64)
    xaty = 0.0
    for t in range(nt):
        for p in range(xv.shape[1]):
            xaty += srcs[t, p] * xv[t, p]
    degenerate = axy == 0.0 and xaty == 0.0
    return AdjointTestResult(axy, xaty, axy - xaty, math.nan if degenerate else axy / xaty,
                             degenerate)


def adjoint_test(model: AcousticModel, seed=7, **kw) -> AdjointTestResult:
    ns = len(model.src_coords or model.default_src())
    nr = len(model.rec_coords or model.default_rec())
    draws = _mt19937_64_uniform(seed, model.nt * (ns + nr), -1.0, 1.0)
    x = draws[: model.nt * ns]
    y = draws[model.nt * ns:]
    return adjoint_test_with(model, x, y, **kw)


# ---------------------------------------------------------------------------
# diffusion application (diffusion.hpp:13-51)

@dataclass
class DiffusionConfig:
    nx: int = 64
    ny: int = 64
    alpha: Fraction = Fraction(1)
    dx: Fraction = Fraction(1)
    dy: Fraction = Fraction(1)
    nt: int = 10
    order: int = 2

    def dt(self) -> Fraction:
        dx2, dy2 = self.dx * self.dx, self.dy * self.dy
        base = dx2 * dy2 / (2 * self.alpha * (dx2 + dy2))
        if self.order == 2:
            return base
        from .fd import fd_weights2
        lam = sum(abs(w) for w in fd_weights2(self.order))
        ratio = Fraction(4) / lam
        return base * ratio if ratio < 1 else base


@dataclass
class DiffusionBuild:
    grid: Grid
    u: GridFunction
    op: Operator


def make_diffusion_operator(cfg: DiffusionConfig, device=0, pinned=False) -> DiffusionBuild:
    if cfg.dx != cfg.dy:
        raise InvalidShapeError("shared spacing symbol requires dx == dy")
    grid = Grid(pinned=pinned)
    u = grid.create_time("u", (cfg.nx, cfg.ny), 1, cfg.order)
    a, d = Fraction(cfg.alpha), Fraction(cfg.dx)
    desc = _lib.DiffusionDesc(cfg.nx, cfg.ny, cfg.order, cfg.nt, a.numerator, a.denominator,
                              d.numerator, d.denominator)
    plan = C.c_void_p()
    check(lib.sf_diffusion_plan_create(C.byref(desc), device, C.byref(plan)))
    return DiffusionBuild(grid, u, Operator(plan.value, [u]))


def diffusion_run(cfg: DiffusionConfig, u0, device=0) -> np.ndarray:
    """Both slots start from u0; returns slot nt % 2 as doubles
    (diffusion.cpp:115-140)."""
    b = make_diffusion_operator(cfg, device)
    u0 = np.asarray(u0, np.float64).reshape(cfg.nx, cfg.ny)
    b.u.data[0] = u0.astype(np.float32)
    b.u.data[1] = u0.astype(np.float32)
    b.op.apply()
    return b.u.data[cfg.nt % 2].astype(np.float64)


def hot_cell_field(nx, ny):
    u = np.zeros((nx, ny))
    u[nx // 2, ny // 2] = 1.0
    return u


def gaussian_blob_field(nx, ny, seed=0):
    """diffusion.cpp:146-163."""
    u = np.zeros((nx, ny))
    cx = nx / 2.0 + (seed % 3)
    cy = ny / 2.0 - (seed % 5)
    w = min(nx, ny) / 12.0
    i = np.arange(nx, dtype=np.float64)[:, None]
    j = np.arange(ny, dtype=np.float64)[None, :]
    dx = (i - cx) / w
    dy = (j - cy) / w
    r2 = dx * dx + dy * dy
    return np.where(r2 < 9.0, np.exp(-r2), 0.0)


# ---------------------------------------------------------------------------
# FWI gradient (config 5; absent from the reference — SPEC.md:635,639)

class FwiPlan:
    """Forward with the full wavefield history in HBM, then the adjoint sweep
    fused with grad += u(t) * v_tt(t)."""

    def __init__(self, shape, space_order, nt, dt, spacing, n_src, n_rec, device=0, pinned=False):
        """pinned: keep page-locked host buffers for the outputs (reused by
        every gradient() call, so copy what must outlive the next call)."""
        self._pinned = pinned
        self._out = {}
        desc = _lib.AcousticDesc()
        desc.ndim = 3
        for i, e in enumerate(shape):
            desc.shape[i] = e
        desc.space_order = space_order
        desc.forward = 1
        desc.nt = nt
        desc.dt = dt
        desc.spacing = spacing
        desc.n_src = n_src
        desc.n_rec = n_rec
        plan = C.c_void_p()
        check(lib.sf_fwi_plan_create(C.byref(desc), device, C.byref(plan)))
        self._plan = plan
        self.shape, self.nt, self.n_src, self.n_rec = tuple(shape), nt, n_src, n_rec

    def __del__(self):
        try:
            lib.sf_plan_destroy(self._plan)
        except Exception:
            pass

    def eta_skip_fraction(self):
        """Forward sweep: fraction of point updates whose eta box is skipped."""
        f = C.c_double()
        check(lib.sf_plan_eta_skip_fraction(self._plan, C.byref(f)))
        return f.value

    def gradient(self, m, eta, src, src_ci, src_w, rec_ci, rec_w, residual, want_v=False,
                 want_src=False):
        f32 = lambda a: np.ascontiguousarray(a, np.float32)  # noqa: E731
        i32 = lambda a: np.ascontiguousarray(a, np.int32)  # noqa: E731
        ins = [f32(m), f32(eta), f32(src), i32(src_ci), f32(src_w), i32(rec_ci), f32(rec_w),
               f32(residual)]
        # the C side reads the plan's full extents from every buffer: check
        # sizes here (InvalidShapeError, as Operator._argv does)
        want = [("m", self.shape), ("eta", self.shape), ("src", (self.nt, self.n_src)),
                ("src_ci", (self.n_src, 3)), ("src_w", (self.n_src, 8)),
                ("rec_ci", (self.n_rec, 3)), ("rec_w", (self.n_rec, 8)),
                ("residual", (self.nt, self.n_rec))]
        for a, (name, shp) in zip(ins, want):
            if a.size != int(np.prod(shp)):
                raise InvalidShapeError(f"{name} must have {int(np.prod(shp))} elements "
                                        f"{shp}, got {a.size}")
        rec_out = self._host("rec_out", (self.nt, self.n_rec))
        grad = self._host("grad", self.shape)
        v = self._host("v", (3,) + self.shape) if want_v else None
        srcs = self._host("srcs", (self.nt, self.n_src)) if want_src else None
        check(lib.sf_fwi_gradient(self._plan, *[a.ctypes.data for a in ins], rec_out.ctypes.data,
                                  grad.ctypes.data, _lib.ptr(v), _lib.ptr(srcs)))
        return rec_out, grad, v, srcs

    def _host(self, name, shape):
        if not self._pinned:
            return np.zeros(shape, np.float32)
        if name not in self._out:
            self._out[name] = pinned_array(shape, np.float32)
        return self._out[name]

    def time(self):
        f = C.c_float()
        a = C.c_float()
        check(lib.sf_fwi_time(self._plan, C.byref(f), C.byref(a)))
        return f.value, a.value

"""ctypes bindings to the CPU checkers in oracle/_ref/.

TEST INFRASTRUCTURE ONLY: used by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference leg. Never imported by the product
package (paper_1609_03361_b200/).

* ``Port`` wraps ``libsf_port.so``: the plain-C restatement (oracle/sf_port.c).
* ``Ref`` wraps ``libsf_ref.so``: the unmodified reference library
  (stencilforge, built from /root/reference/proj/src by oracle/Makefile) driven
  through its public API (oracle/ref_driver.cpp).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_DIR = os.path.join(ROOT, "oracle", "_ref")

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")


class SfpRat(C.Structure):
    _fields_ = [("num", C.c_int64), ("den", C.c_int64)]


class SfpAcousticCoefs(C.Structure):
    _fields_ = [
        ("ndim", C.c_int), ("order", C.c_int), ("forward", C.c_int),
        ("ce", C.c_float), ("cm", C.c_float),
        ("tc", C.c_float * 3), ("tfield", C.c_int * 3), ("tlevel", C.c_int * 3),
        ("c0", C.c_float), ("cj", C.c_float * 8), ("src_scale", C.c_float),
    ]


def _load(name):
    path = os.path.join(REF_DIR, name)
    if not os.path.exists(path):
        return None
    return C.CDLL(path)


class Port:
    """The C restatement of the generated kernels (oracle/sf_port.c)."""

    def __init__(self):
        lib = _load("libsf_port.so")
        if lib is None:
            raise RuntimeError("oracle/_ref/libsf_port.so missing: run make -C oracle")
        self.lib = lib
        lib.sfp_fd_weights2.argtypes = [C.c_int, C.POINTER(SfpRat)]
        lib.sfp_make_acoustic_coefs.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double,
                                                C.c_double, C.POINTER(SfpAcousticCoefs)]
        lib.sfp_stable_dt.restype = C.c_double
        lib.sfp_stable_dt.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, C.c_double]
        lib.sfp_ricker.restype = C.c_double
        lib.sfp_ricker.argtypes = [C.c_double] * 3
        lib.sfp_interp_weights.argtypes = [C.c_int, _f64p, C.c_double, _i64p, _i32p, _f32p]
        lib.sfp_build_medium.argtypes = [C.c_int, _i64p, C.c_int, C.c_double, C.c_double,
                                         C.c_double, _f32p, _f32p]
        lib.sfp_medium_from_velocity.argtypes = [C.c_int, _i64p, C.c_int, C.c_double,
                                                 C.c_double, _f64p, _f32p, _f32p]
        lib.sfp_acoustic_run.argtypes = [C.POINTER(SfpAcousticCoefs), _i64p, C.c_int64, _f32p,
                                         _f32p, _f32p, _f32p, _i32p, _f32p, C.c_int64, _f32p,
                                         _i32p, _f32p, C.c_int64, C.c_int]
        lib.sfp_acoustic_forward_history.argtypes = lib.sfp_acoustic_run.argtypes
        lib.sfp_fwi_adjoint_gradient.argtypes = [
            C.POINTER(SfpAcousticCoefs), _i64p, C.c_int64, _f32p, _f32p, _f32p, _f32p,
            _f32p, _i32p, _f32p, C.c_int64, _f32p, _i32p, _f32p, C.c_int64, _f32p, C.c_int]
        lib.sfp_smooth_taps.argtypes = [C.c_double, _f64p]
        lib.sfp_smooth_extrema.argtypes = [_i64p, C.c_int64, C.c_int64, C.c_uint64, C.c_double,
                                           C.POINTER(C.c_double), C.POINTER(C.c_double)]
        lib.sfp_smooth_medium.argtypes = [_i64p, C.c_int64, C.c_int64, C.c_uint64, C.c_double,
                                          C.c_double, C.c_double, C.c_int, C.c_double, C.c_double,
                                          C.c_double, C.c_double, _f32p, _f32p]
        lib.sfp_diffusion_coefs.argtypes = [SfpRat, SfpRat, C.c_int, C.POINTER(C.c_float),
                                            C.POINTER(C.c_int), C.POINTER(C.c_float)]
        lib.sfp_diffusion_dt.argtypes = [SfpRat, SfpRat, C.c_int, C.POINTER(SfpRat)]
        lib.sfp_diffusion_run.argtypes = [C.c_int64, C.c_int64, C.c_int, C.c_float, C.c_int,
                                          C.POINTER(C.c_float), C.c_int64, _f32p, C.c_int]

    # -- setup -------------------------------------------------------------
    def fd_weights2(self, order):
        w = (SfpRat * (order + 1))()
        assert self.lib.sfp_fd_weights2(order, w) == 0
        return [(x.num, x.den) for x in w]

    def coefs(self, ndim, order, forward, dt, spacing):
        c = SfpAcousticCoefs()
        assert self.lib.sfp_make_acoustic_coefs(ndim, order, int(forward), dt, spacing,
                                                C.byref(c)) == 0
        return c

    def stable_dt(self, ndim, order, spacing, v_top, v_bottom):
        return self.lib.sfp_stable_dt(ndim, order, spacing, v_top, v_bottom)

    def ricker(self, f0, t, t0):
        return self.lib.sfp_ricker(f0, t, t0)

    def interp(self, coords, spacing, extents):
        coords = np.ascontiguousarray(coords, np.float64)
        ndim = coords.shape[1]
        ext = np.asarray(extents, np.int64)
        ci = np.zeros((len(coords), ndim), np.int32)
        w = np.zeros((len(coords), 1 << ndim), np.float32)
        for p in range(len(coords)):
            rc = self.lib.sfp_interp_weights(ndim, coords[p].copy(), spacing, ext, ci[p], w[p])
            if rc != 0:
                raise ValueError(f"OutOfDomainError: point {p}")
        return ci, w

    def medium(self, shape, boundary_width, spacing, v_top, v_bottom):
        shape = np.asarray(shape, np.int64)
        m = np.zeros(tuple(shape), np.float32)
        eta = np.zeros(tuple(shape), np.float32)
        self.lib.sfp_build_medium(len(shape), shape, boundary_width, spacing, v_top,
                                  v_bottom, m.reshape(-1), eta.reshape(-1))
        return m, eta

    def medium_from_velocity(self, v, boundary_width, spacing, v_min):
        shape = np.asarray(v.shape, np.int64)
        m = np.zeros(v.shape, np.float32)
        eta = np.zeros(v.shape, np.float32)
        self.lib.sfp_medium_from_velocity(len(shape), shape, boundary_width, spacing, v_min,
                                          np.ascontiguousarray(v, np.float64).reshape(-1),
                                          m.reshape(-1), eta.reshape(-1))
        return m, eta

    def smooth_extrema(self, shape, b, e, seed, sigma=8.0):
        lo, hi = C.c_double(), C.c_double()
        rc = self.lib.sfp_smooth_extrema(np.asarray(shape, np.int64), b, e, seed, sigma,
                                         C.byref(lo), C.byref(hi))
        assert rc == 0, rc
        return lo.value, hi.value

    def smooth_medium(self, shape, b, e, seed, lo, hi, sigma=8.0, v_lo=1500.0, v_hi=4500.0,
                      boundary_width=40, spacing=10.0, v_min=1500.0):
        """m, eta of global planes [b, e) (csrc/medium.cu's definition)."""
        out = (e - b, shape[1], shape[2])
        m = np.zeros(out, np.float32)
        eta = np.zeros(out, np.float32)
        rc = self.lib.sfp_smooth_medium(np.asarray(shape, np.int64), b, e, seed, sigma, v_lo,
                                        v_hi, boundary_width, spacing, v_min, lo, hi,
                                        m.reshape(-1), eta.reshape(-1))
        assert rc == 0, rc
        return m, eta

    # -- runs --------------------------------------------------------------
    def acoustic_run(self, coefs, u, m, eta, inj, inj_ci, inj_w, smp, smp_ci, smp_w, nt,
                     nthreads=0):
        shape = np.asarray(m.shape, np.int64)
        rc = self.lib.sfp_acoustic_run(C.byref(coefs), shape, nt, u.reshape(-1),
                                       m.reshape(-1), eta.reshape(-1), inj.reshape(-1),
                                       inj_ci.reshape(-1), inj_w.reshape(-1), inj_ci.shape[0],
                                       smp.reshape(-1), smp_ci.reshape(-1), smp_w.reshape(-1),
                                       smp_ci.shape[0], nthreads)
        assert rc == 0

    def forward_history(self, coefs, hist, m, eta, src, src_ci, src_w, rec, rec_ci, rec_w,
                        nt, nthreads=0):
        shape = np.asarray(m.shape, np.int64)
        rc = self.lib.sfp_acoustic_forward_history(
            C.byref(coefs), shape, nt, hist.reshape(-1), m.reshape(-1), eta.reshape(-1),
            src.reshape(-1), src_ci.reshape(-1), src_w.reshape(-1), src_ci.shape[0],
            rec.reshape(-1), rec_ci.reshape(-1), rec_w.reshape(-1), rec_ci.shape[0], nthreads)
        assert rc == 0

    def adjoint_gradient(self, coefs, v, m, eta, hist, rec, rec_ci, rec_w, src, src_ci, src_w,
                         grad, nt, nthreads=0):
        shape = np.asarray(m.shape, np.int64)
        rc = self.lib.sfp_fwi_adjoint_gradient(
            C.byref(coefs), shape, nt, v.reshape(-1), m.reshape(-1), eta.reshape(-1),
            hist.reshape(-1), rec.reshape(-1), rec_ci.reshape(-1), rec_w.reshape(-1),
            rec_ci.shape[0], src.reshape(-1), src_ci.reshape(-1), src_w.reshape(-1),
            src_ci.shape[0], grad.reshape(-1), nthreads)
        assert rc == 0

    def diffusion_coefs(self, alpha, dx, order):
        c0 = C.c_float()
        has = C.c_int()
        cj = (C.c_float * 8)()
        assert self.lib.sfp_diffusion_coefs(SfpRat(*alpha), SfpRat(*dx), order, C.byref(c0),
                                            C.byref(has), cj) == 0
        return c0.value, bool(has.value), list(cj)

    def diffusion_run(self, u, order, alpha, dx, nt, nthreads=0):
        """u: (2, nx, ny) float32, both slots initialised; returns final slot."""
        c0, has, cj = self.diffusion_coefs(alpha, dx, order)
        cjarr = (C.c_float * 8)(*cj)
        nx, ny = u.shape[1:]
        assert self.lib.sfp_diffusion_run(nx, ny, order, c0, int(has), cjarr, nt,
                                          u.reshape(-1), nthreads) == 0
        return u[nt % 2]


class Ref:
    """The reference library itself (oracle/_ref/libsf_ref.so)."""

    def __init__(self):
        lib = _load("libsf_ref.so")
        if lib is None:
            raise RuntimeError("oracle/_ref/libsf_ref.so missing (reference not built)")
        self.lib = lib
        lib.sfref_last_error.restype = C.c_char_p
        lib.sfref_acoustic_build.restype = C.c_void_p
        lib.sfref_acoustic_build.argtypes = [
            C.c_int, _i64p, C.c_int, C.c_double, C.c_long, C.c_double, C.c_int, C.c_double,
            C.c_double, C.c_double, C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_int]
        lib.sfref_acoustic_stable_dt.restype = C.c_double
        lib.sfref_acoustic_stable_dt.argtypes = [C.c_int, _i64p, C.c_double, C.c_int,
                                                 C.c_double, C.c_double]
        lib.sfref_ricker.restype = C.c_double
        lib.sfref_ricker.argtypes = [C.c_double] * 3
        lib.sfref_diffusion_build.restype = C.c_void_p
        lib.sfref_diffusion_build.argtypes = [C.c_long] * 7 + [C.c_int]
        lib.sfref_free.argtypes = [C.c_void_p]
        lib.sfref_dt.restype = C.c_double
        lib.sfref_dt.argtypes = [C.c_void_p]
        lib.sfref_buffer_bytes.restype = C.c_long
        lib.sfref_buffer_bytes.argtypes = [C.c_void_p, C.c_char_p]
        lib.sfref_get.argtypes = [C.c_void_p, C.c_char_p, C.c_void_p, C.c_long]
        lib.sfref_set.argtypes = [C.c_void_p, C.c_char_p, C.c_void_p, C.c_long]
        lib.sfref_build.argtypes = [C.c_void_p]
        lib.sfref_apply.argtypes = [C.c_void_p]
        lib.sfref_source.restype = C.c_char_p
        lib.sfref_source.argtypes = [C.c_void_p]
        lib.sfref_nest.restype = C.c_char_p
        lib.sfref_nest.argtypes = [C.c_void_p]
        lib.sfref_interp_weights.argtypes = [C.c_int, _f64p, C.c_double, _i64p,
                                             C.POINTER(C.c_long), _f64p]
        lib.sfref_set_threads.argtypes = [C.c_int]
        lib.sfref_set_blocking.argtypes = [C.c_int, C.POINTER(C.c_long)]

    def set_blocking(self, sizes=()):
        """Blocking plan (x, y, z sizes; 0 = unblocked) for the next builds."""
        arr = (C.c_long * 3)(*(list(sizes) + [0] * (3 - len(sizes))))
        self.lib.sfref_set_blocking(3, arr)

    def error(self):
        return self.lib.sfref_last_error().decode()

    def set_threads(self, n):
        self.lib.sfref_set_threads(n)

    def max_threads(self):
        return self.lib.sfref_max_threads()


class RefOperator:
    """A built reference operator (acoustic or diffusion) and its grid."""

    def __init__(self, ref: Ref, handle):
        self.ref = ref
        self.h = handle

    def __del__(self):
        try:
            self.ref.lib.sfref_free(self.h)
        except Exception:
            pass

    @property
    def dt(self):
        return self.ref.lib.sfref_dt(self.h)

    def get(self, name, dtype, shape):
        arr = np.empty(shape, dtype)
        n = self.ref.lib.sfref_buffer_bytes(self.h, name.encode())
        assert n == arr.nbytes, (name, n, arr.nbytes)
        assert self.ref.lib.sfref_get(self.h, name.encode(), arr.ctypes.data, arr.nbytes) == 0
        return arr

    def set(self, name, arr):
        arr = np.ascontiguousarray(arr)
        assert self.ref.lib.sfref_set(self.h, name.encode(), arr.ctypes.data, arr.nbytes) == 0, \
            self.ref.error()

    def build(self):
        assert self.ref.lib.sfref_build(self.h) == 0, self.ref.error()

    def apply(self):
        rc = self.ref.lib.sfref_apply(self.h)
        assert rc == 0, self.ref.error()

    def source(self):
        s = self.ref.lib.sfref_source(self.h)
        assert s is not None, self.ref.error()
        return s.decode()

    def nest(self):
        s = self.ref.lib.sfref_nest(self.h)
        assert s is not None, self.ref.error()
        return s.decode()


@dataclass
class AcousticCase:
    """Mirror of sf::AcousticModel (acoustic.hpp:17-42) for test setups."""
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


def ref_acoustic(ref: Ref, case: AcousticCase, forward: bool) -> RefOperator:
    shape = np.asarray(case.shape, np.int64)
    ndim = len(case.shape)
    src = np.ascontiguousarray(case.src_coords, np.float64).reshape(-1)
    rec = np.ascontiguousarray(case.rec_coords, np.float64).reshape(-1)
    h = ref.lib.sfref_acoustic_build(
        ndim, shape, case.boundary_width, case.spacing, case.nt, case.dt, case.space_order,
        case.f0, case.v_top, case.v_bottom, len(case.src_coords),
        src.ctypes.data if len(src) else None, len(case.rec_coords),
        rec.ctypes.data if len(rec) else None, int(forward))
    if not h:
        raise RuntimeError(ref.error())
    op = RefOperator(ref, h)
    op._keep = (src, rec)
    return op


def ref_diffusion(ref: Ref, nx, ny, alpha, dx, nt, order) -> RefOperator:
    h = ref.lib.sfref_diffusion_build(nx, ny, alpha[0], alpha[1], dx[0], dx[1], nt, order)
    if not h:
        raise RuntimeError(ref.error())
    return RefOperator(ref, h)


def have_ref() -> bool:
    return os.path.exists(os.path.join(REF_DIR, "libsf_ref.so"))


def have_port() -> bool:
    return os.path.exists(os.path.join(REF_DIR, "libsf_port.so"))

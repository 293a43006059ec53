"""ctypes binding of libsf_b200.so (C ABI: include/sf_b200.h).

The shared library is built in-tree by ``make -C paper_1609_03361_b200/csrc``
(``__graft_entry__.build()``). There is no CPU fallback: importing this module
without the library raises, and every plan constructor fails loudly without a
sm_100 device.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsf_b200.so")

SF_OK = 0
SF_ERR_INVALID = 1
SF_ERR_CFL = 2
SF_ERR_OUT_OF_DOMAIN = 3
SF_ERR_SIGNATURE = 4
SF_ERR_KERNEL = 5
SF_ERR_CUDA = 6
SF_ERR_OOM = 7

# header-declared entry points (include/sf_b200.h); tests check every one is
# exported by the built library
EXPORTS = [
    "sf_last_error", "sf_device_count",
    "sf_acoustic_plan_create", "sf_diffusion_plan_create", "sf_plan_destroy",
    "sf_acoustic_plan_create_ex", "sf_diffusion_plan_create_ex",
    "sf_plan_num_args", "sf_plan_arg_name", "sf_plan_arg_bytes",
    "sf_acoustic_apply", "sf_diffusion_apply", "sf_plan_invoke",
    "sf_plan_upload", "sf_plan_run", "sf_plan_download", "sf_plan_synchronize",
    "sf_plan_time",
    "sf_fwi_plan_create", "sf_fwi_gradient", "sf_fwi_time",
    "sf_interpolation_weights", "sf_stable_dt", "sf_ricker", "sf_build_medium",
    "sf_acoustic_constants", "sf_diffusion_constants",
    "sf_acoustic_plan_create_slab", "sf_slab_chain_run", "sf_nccl_unique_id",
    "sf_plan_attach_nccl", "sf_plan_autotune", "sf_plan_save_buffer", "sf_plan_load_buffer",
    "sf_plan_dump_csv", "sf_plan_save_series_text", "sf_selftest_reciprocal",
    "sf_plan_eta_skip_fraction", "sf_smooth_extrema", "sf_smooth_medium",
    "sf_plan_set_smooth_medium",
]


class AcousticDesc(C.Structure):
    _fields_ = [
        ("ndim", C.c_int), ("shape", C.c_int64 * 3), ("space_order", C.c_int),
        ("forward", C.c_int), ("nt", C.c_int64), ("dt", C.c_double),
        ("spacing", C.c_double), ("n_src", C.c_int64), ("n_rec", C.c_int64),
    ]


class DiffusionDesc(C.Structure):
    _fields_ = [
        ("nx", C.c_int64), ("ny", C.c_int64), ("order", C.c_int), ("nt", C.c_int64),
        ("alpha_num", C.c_int64), ("alpha_den", C.c_int64),
        ("dx_num", C.c_int64), ("dx_den", C.c_int64),
    ]


class TuneEntry(C.Structure):
    _fields_ = [("kind", C.c_int), ("tile_nx", C.c_int), ("tile_ty", C.c_int),
                ("vec_warps", C.c_int), ("stages", C.c_int), ("median_ms", C.c_float)]


class SlabDesc(C.Structure):
    _fields_ = [("global_n0", C.c_int64), ("plane0", C.c_int64), ("own_begin", C.c_int64),
                ("own_end", C.c_int64)]


class SmoothMediumDesc(C.Structure):
    _fields_ = [("shape", C.c_int64 * 3), ("a0_begin", C.c_int64), ("a0_end", C.c_int64),
                ("seed", C.c_uint64), ("sigma", C.c_double), ("v_lo", C.c_double),
                ("v_hi", C.c_double), ("boundary_width", C.c_int), ("spacing", C.c_double),
                ("v_min", C.c_double)]


_vp = C.c_void_p
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")


def _bind(lib):
    lib.sf_last_error.restype = C.c_char_p
    lib.sf_device_count.restype = C.c_int
    lib.sf_acoustic_plan_create.argtypes = [C.POINTER(AcousticDesc), C.c_int, C.POINTER(_vp)]
    lib.sf_diffusion_plan_create.argtypes = [C.POINTER(DiffusionDesc), C.c_int, C.POINTER(_vp)]
    lib.sf_fwi_plan_create.argtypes = [C.POINTER(AcousticDesc), C.c_int, C.POINTER(_vp)]
    lib.sf_plan_destroy.argtypes = [_vp]
    lib.sf_plan_destroy.restype = None
    lib.sf_plan_num_args.argtypes = [_vp]
    lib.sf_plan_arg_name.argtypes = [_vp, C.c_int]
    lib.sf_plan_arg_name.restype = C.c_char_p
    lib.sf_plan_arg_bytes.argtypes = [_vp, C.c_int]
    lib.sf_plan_arg_bytes.restype = C.c_int64
    lib.sf_acoustic_apply.argtypes = [_vp] * 10
    lib.sf_diffusion_apply.argtypes = [_vp, _vp]
    lib.sf_plan_invoke.argtypes = [_vp, C.POINTER(_vp), C.c_int]
    lib.sf_plan_upload.argtypes = [_vp, C.POINTER(_vp), C.c_int]
    lib.sf_plan_download.argtypes = [_vp, C.POINTER(_vp), C.c_int]
    lib.sf_plan_run.argtypes = [_vp, C.c_int64, C.c_int64]
    lib.sf_plan_synchronize.argtypes = [_vp]
    lib.sf_plan_time.argtypes = [_vp, C.POINTER(C.c_float), C.POINTER(C.c_float),
                                 C.POINTER(C.c_int64)]
    lib.sf_fwi_gradient.argtypes = [_vp] * 13
    lib.sf_fwi_time.argtypes = [_vp, C.POINTER(C.c_float), C.POINTER(C.c_float)]
    lib.sf_interpolation_weights.argtypes = [C.c_int, _f64p, C.c_double, _i64p, _i32p, _f32p]
    lib.sf_stable_dt.restype = C.c_double
    lib.sf_stable_dt.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, C.c_double]
    lib.sf_ricker.restype = C.c_double
    lib.sf_ricker.argtypes = [C.c_double, C.c_double, C.c_double]
    lib.sf_build_medium.argtypes = [C.c_int, _i64p, C.c_int, C.c_double, C.c_double, C.c_double,
                                    _vp, C.c_double, _f32p, _f32p]
    lib.sf_acoustic_constants.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                          _f32p, _i32p]
    lib.sf_acoustic_plan_create_ex.argtypes = [C.POINTER(AcousticDesc), _f32p, _i32p, C.c_int,
                                               C.POINTER(_vp)]
    lib.sf_diffusion_plan_create_ex.argtypes = [C.POINTER(DiffusionDesc), C.c_float, C.c_int,
                                                _f32p, C.c_int, C.POINTER(_vp)]
    lib.sf_diffusion_constants.argtypes = [C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_int64,
                                           C.POINTER(C.c_float), C.POINTER(C.c_int), _f32p]
    lib.sf_acoustic_plan_create_slab.argtypes = [C.POINTER(AcousticDesc), C.POINTER(SlabDesc),
                                                 C.c_int, C.POINTER(_vp)]
    lib.sf_slab_chain_run.argtypes = [C.POINTER(_vp), C.c_int, C.c_int64, C.c_int64]
    lib.sf_nccl_unique_id.argtypes = [C.c_char_p, C.c_int]
    lib.sf_plan_attach_nccl.argtypes = [_vp, C.c_char_p, C.c_int, C.c_int]
    lib.sf_plan_save_buffer.argtypes = [_vp, C.c_char_p, C.c_char_p]
    lib.sf_plan_load_buffer.argtypes = [_vp, C.c_char_p, C.c_char_p]
    lib.sf_plan_dump_csv.argtypes = [_vp, C.c_char_p, C.c_char_p, C.c_long]
    lib.sf_plan_save_series_text.argtypes = [_vp, C.c_char_p, C.c_char_p]
    lib.sf_selftest_reciprocal.argtypes = [C.c_int, C.POINTER(C.c_ulonglong)]
    lib.sf_plan_eta_skip_fraction.argtypes = [_vp, C.POINTER(C.c_double)]
    lib.sf_plan_autotune.argtypes = [_vp, C.c_int64, C.c_int, C.POINTER(TuneEntry), C.c_int,
                                     C.POINTER(C.c_int)]
    lib.sf_smooth_extrema.argtypes = [C.POINTER(SmoothMediumDesc), C.c_int,
                                      C.POINTER(C.c_double), C.POINTER(C.c_double)]
    lib.sf_smooth_medium.argtypes = [C.POINTER(SmoothMediumDesc), C.c_double, C.c_double,
                                     C.c_int, _vp, _vp]
    lib.sf_plan_set_smooth_medium.argtypes = [_vp, C.POINTER(SmoothMediumDesc), C.c_double,
                                              C.c_double]
    return lib


def load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `make -C paper_1609_03361_b200/csrc` "
            "(the B200 path has no CPU fallback)")
    return _bind(C.CDLL(LIB_PATH))


lib = load()


def last_error() -> str:
    return lib.sf_last_error().decode(errors="replace")


def ptr(a) -> int | None:
    """Raw data pointer of a numpy array (None passes through)."""
    if a is None:
        return None
    return a.ctypes.data

"""B200-native stencil hot path of the Devito-style finite-difference toolkit
(reference: stencilforge, arXiv 1609.03361).

The product is ``libsf_b200.so`` (CUDA kernels for sm_100a + C++ host code,
C ABI in include/sf_b200.h). This package binds it and mirrors the
reference's public API (``api``). Importing fails loudly if the library has
not been built: there is no CPU fallback.
"""
from . import _lib  # noqa: F401  (raises ImportError when the .so is missing)
from .api import (  # noqa: F401
    AcousticModel, AcousticSetup, AdjointTestResult, CflViolationError, CudaError,
    DiffusionConfig, FwiPlan, Grid, GridFunction, InvalidOrderError, InvalidShapeError,
    KernelFailedError, Operator, OutOfDomainError, SfError, SignatureMismatchError,
    SmoothMedium, SparsePointSet, acoustic_adjoint, acoustic_build, acoustic_forward, adjoint_test,
    adjoint_test_with, build_medium, diffusion_run, gaussian_blob_field, hot_cell_field,
    interpolation_weights, load_series_column, make_diffusion_operator, ricker_wavelet,
)

LIB_PATH = _lib.LIB_PATH

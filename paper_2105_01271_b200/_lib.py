"""ctypes binding of the device library (include/sketchpress_b200.h).

This is exactly the binding a maintainer of the reference would add
(INTEGRATION.md): plain pointers, sizes and a cudaStream_t, an int status that
maps onto the reference's exception classes (src/errors.py), warning bits
returned through an ``info`` array.

There is no CPU fallback: importing the compute entry points without the
built library or without a CUDA device raises immediately.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

from .errors import ConfigError, FormatError, NumericalError, SketchpressError

LIB_PATH = Path(__file__).resolve().parent / "libsketchpress_b200.so"

SP_OK, SP_ECONFIG, SP_EIO, SP_ENUMERICAL, SP_ECUDA = 0, 2, 3, 4, 5
SP_F64, SP_F32 = 0, 1
SP_WARN_RANK_DEFICIENT, SP_WARN_LIFT_CLAMPED, SP_WARN_ID_PINV, SP_WARN_BULK_SPLIT = 1, 2, 4, 8
SP_HINT_COLS_VALIDATED, SP_HINT_SAME_SET, SP_HINT_DIFFERENT_SET = 1, 2, 4
INFO_KEPT, INFO_WARN, INFO_BLOCK, INFO_ITERS, INFO_RANK, INFO_LIFT_R, INFO_LAUNCHES, INFO_FUSED = range(8)
INFO_LEN = 8

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int32
_D = ctypes.c_double

# name -> argtypes (restype is int status unless listed in _RESTYPES)
SIGNATURES = {
    "sp_abi_version": [],
    "sp_last_error": [],
    "sp_launch_count": [],
    "sp_release_workspaces": [],
    "sp_deferred_status": [_P],
    "sp_set_finish_mode": [_I32],
    "sp_apply_stencil": [_P, _I32, _I64, _I64, _I64, _P, _P, _I32, _I64, _I32, _P, _I64, _P],
    "sp_check_columns": [_P, _I64, _I64, _P],
    "sp_skinny_atz": [_P, _I32, _I64, _I64, _I64, _P, _I64, _I32, _P, _I64, _P],
    "sp_gemm": [_I32, _I32, _I64, _I64, _I64, _D, _P, _I64, _P, _I64, _D, _P, _I64, _P],
    "sp_gemm_aat": [_I64, _I64, _P, _I64, _P, _I64, _P],
    "sp_gemm_exact": [_I32, _I64, _I64, _I64, _P, _I64, _P, _P, _I64, _P, _P, _I64, _P],
    "sp_exact_plan": [_I64, _P, _P],
    "sp_exponents": [_I32, _I64, _I64, _P, _I64, _P, _P],
    "sp_gemm_exact_levels": [_I32, _I64, _I64, _I64, _P, _I64, _P, _P, _I64, _P, _I32, _I32, _P, _P],
    "sp_dd_levels": [_I64, _I64, _P, _I32, _P, _P, _P, _I64, _P],
    "sp_pqd_begin": [_I64, _I64, _I32, _P, _I64, _P, _P, _P, _I64, _P, _P],
    "sp_pqd_select": [_I32, _I32, _I64, _I64, _P, _P, _P, _I64, _P, _P, _P, _P, _P],
    "sp_pqd_orth": [_I32, _I64, _P, _P, _I64, _P, _P, _P, _P],
    "sp_pqd_coef": [_I32, _I64, _I64, _P, _P, _I64, _P, _P, _P, _P, _P],
    "sp_pqd_update": [_I32, _I64, _I64, _P, _P, _I64, _P, _P, _P, _P],
    "sp_id_from_qr": [_I64, _I32, _P, _P, _I64, _P, _P, _P, _P],
    "sp_tsqr": [_I64, _I64, _P, _I64, _P, _I64, _P, _I64, _P],
    "sp_qr_tall": [_I64, _I64, _P, _I64, _P, _I64, _P, _I64, _I32, _P],
    "sp_cholqr2_async": [_I64, _I64, _P, _I64, _P, _I64, _P, _I64, _P, _P],
    "sp_thin_qr": [_I64, _I64, _P, _I64, _P, _I64, _P, _I64, _P],
    "sp_jacobi_svd": [_I64, _P, _I64, _P, _I64, _P, _P, _I64, _P],
    "sp_thin_svd": [_I64, _I64, _P, _I64, _P, _I64, _P, _P, _I64, _P],
    "sp_thin_svd_t": [_I64, _I64, _P, _I64, _P, _I64, _P, _P, _I64, _P],
    "sp_scale_columns": [_I64, _I64, _P, _I64, _P, _I32, _P],
    "sp_gather_rows": [_P, _I32, _I64, _I64, _P, _I64, _P, _I64, _P],
    "sp_fill_uniform": [_I64, _I64, _P, _I64, ctypes.c_uint64, _I64, _P],
    "sp_pinv_apply": [_P, _I64, _D, _P, _P],
    "sp_trsm_upper": [_I64, _P, _I64, _I64, _P, _I64, _P, _I64, _P],
    "sp_pivoted_qr": [_I64, _I64, _P, _I64, _I32, _P, _P, _I64, _P, _I64, _P],
    "sp_row_id": [_I64, _I64, _P, _I64, _I32, _P, _P, _P, _P],
    "sp_sketch_basis": [_P, _I64, _I64, _I64, _D, _I32, _P, _I64, _P, _P, _P],
    "sp_householder_complete": [_I64, _I32, _I32, _P, _I64, _P, _P],
    "sp_gram_chol_dd": [_I64, _I32, _P, _I64, _P, _I64, _P],
    "sp_srht_sketch": [_I64, _I64, _P, _I64, _I32, ctypes.c_uint64, _P, _I64, _P, _P],
    "sp_srht_gather": [_P, _I32, _I64, _I64, _P, _I64, _P, _I64, _I32, ctypes.c_uint64, _P, _I64, _P, _P],
    "sp_single_pass_svd": [_P, _I32, _I64, _I64, _I64, _P, _P, _I32, _I64, _P, _I64, _I32, _P,
                           _P, _P, _P, _P, _P],
    "sp_power_svd": [_P, _I32, _I64, _I64, _I64, _P, _P, _I32, _I64, _P, _I64, _P, _I64, _I32,
                     _I32, _P, _P, _I32, _P, _P, _P, _P, _P],
    "sp_power_id": [_P, _I32, _I64, _I64, _I64, _P, _P, _I32, _I64, _P, _I64, _I32, _I32, _I32,
                    _P, _I64, _I32, _P, _P, _P, _P, _P, _P, _P, _P, _I32, _P, _P],
    "sp_frob_residual": [_P, _I32, _I64, _I64, _I64, _P, _I64, _P, _P, _I64, _I32, _P, _P],
}
_RESTYPES = {"sp_last_error": ctypes.c_char_p, "sp_launch_count": ctypes.c_int64}

_lib = None


def load():
    """Load (building first if the sources are newer) the device library."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.environ.get("SPB_NO_BUILD"):
        try:
            from .build import build, _stale
            if _stale() and Path("/usr/local/cuda/bin/nvcc").exists():
                build()
        except Exception:  # a prebuilt .so may still be usable; load() reports
            pass
    if not LIB_PATH.exists():
        raise SketchpressError(
            f"device library {LIB_PATH.name} is not built; run `python -m paper_2105_01271_b200.build`")
    lib = ctypes.CDLL(str(LIB_PATH))
    for name, args in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = _RESTYPES.get(name, ctypes.c_int)
    if lib.sp_abi_version() != 1:
        raise SketchpressError("device library ABI mismatch")
    _lib = lib
    return lib


def last_error() -> str:
    msg = load().sp_last_error()
    return msg.decode() if msg else ""


def check(status: int, what: str = "") -> None:
    """Raise the reference's exception class for a non-zero status."""
    if status == SP_OK:
        return
    msg = last_error() or what
    if status == SP_ECONFIG:
        raise ConfigError(msg)
    if status == SP_ENUMERICAL:
        raise NumericalError(msg)
    if status == SP_EIO:
        raise FormatError(msg)
    raise SketchpressError(f"CUDA failure in {what}: {msg}")


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)


def launch_count() -> int:
    return int(load().sp_launch_count())


def release_workspaces() -> None:
    """Return the library's cached workspaces (and the CUDA pool's reserve) to the driver."""
    call("sp_release_workspaces")


def deferred_status() -> int:
    """Flag of this thread's last fused-finish pipeline call (waits for it)."""
    f = ctypes.c_int32(0)
    check(load().sp_deferred_status(ctypes.byref(f)), "sp_deferred_status")
    return int(f.value)


class householder_finish:
    """Context: pipeline calls on this thread use the Householder TSQR finish."""

    def __enter__(self):
        call("sp_set_finish_mode", 1)
        return self

    def __exit__(self, *exc):
        call("sp_set_finish_mode", 0)


def new_info() -> np.ndarray:
    return np.zeros(INFO_LEN, dtype=np.int64)


def info_ptr(info: np.ndarray):
    return info.ctypes.data_as(ctypes.c_void_p)

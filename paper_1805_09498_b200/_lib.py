"""ctypes binding of libffca_b200.so (the C ABI declared in include/ffca.h).

There is no CPU fallback: importing the product modules without the built
library, or calling them without a CUDA device, raises ``BackendUnavailable``.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from .errors import (
    BackendUnavailable,
    DimensionMismatch,
    NotPositiveDefinite,
    SingularP,
    SingularWeightedCovariance,
)

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FFCA_LIB", os.path.join(_HERE, "libffca_b200.so"))

C128, C64 = 0, 1
MEM_HOST, MEM_DEVICE, MEM_HOST_STATS_DEVICE = 0, 1, 2
VF_SCALAR, VF_BIN, VF_FULL, VF_AUTO = 0, 1, 2, 3

OK, E_ARG, E_CUDA, E_SINGULAR_P, E_SINGULAR_B, E_NOT_PD, E_UNSUPPORTED = 0, -1, -2, -3, -4, -5, -6

ST_SINGULAR_P, ST_SINGULAR_B, ST_B_LOADED, ST_NOT_PD, ST_S_LOADED = 1, 2, 4, 8, 16

_vp = ctypes.c_void_p
_i = ctypes.c_int
_d = ctypes.c_double
_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int)

# name -> argtypes (restype int unless listed in _RESTYPES)
SIGNATURES = {
    "ffca_version": [],
    "ffca_last_error": [],
    "ffca_device_count": [],
    "ffca_host_alloc": [ctypes.POINTER(_vp), ctypes.c_longlong],
    "ffca_host_free": [_vp],
    "ffca_last_launch_count": [],
    "ffca_set_kernel_timing": [_i],
    "ffca_last_kernel_ms": [],
    "ffca_plan_loop": [_i, _i, _i, _i, _i, _i, _i, _i, _ip],
    "ffca_plan_loop_ex": [_i, _i, _i, _i, _i, _i, _i, _i, _i, _ip],
    "ffca_fastfca_run": [_i, _vp, _i, _i, _i, _i, _i, _i, _i, _vp, _vp, _vp, _vp, _i, _d, _vp, _i, _i, _i,
                         _vp, _vp, _vp, _vp, _vp, _vp],
    "ffca_fastfca_run_stats": [_i, _vp, _i, _i, _i, _i, _i, _i, _i, _vp, _vp, _vp, _vp, _i, _d, _vp, _i, _i, _i,
                               _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "ffca_fastfca_stats": [_i, _vp, _i, _i, _i, _i, _i, _i, _i, _vp, _vp, _vp, _vp, _vp, _vp],
    "ffca_fastfca_images": [_i, _vp, _i, _i, _i, _i, _i, _i, _i, _vp, _vp, _vp, _vp, _vp, _vp],
    "ffca_back_transform": [_i, _vp, _i, _i, _i, _i, _i, _i, _i, _vp, _vp, _vp, _i, _vp],
    "ffca_fastfca_loglik": [_i, _vp, _i, _i, _i, _i, _i, _i, _i, _vp, _vp, _vp, _vp, _vp, _vp],
    "ffca_fixed_point_update_P": [_i, _vp, _i, _i, _i, _i, _i, _i, _i, _vp, _vp, _vp, _vp, _i, _vp, _vp],
    "ffca_fca_run": [_i, _vp, _i, _i, _i, _i, _i, _i, _i, _vp, _vp, _vp, _i, _d, _vp, _i, _i, _vp, _vp, _vp,
                     _vp, _vp, _vp],
    "ffca_fca_estep": [_i, _vp, _i, _i, _i, _i, _i, _i, _i, _vp, _vp, _vp, _vp, _vp, _i, _vp],
    "ffca_fca_loglik": [_i, _vp, _i, _i, _i, _i, _i, _i, _i, _vp, _vp, _vp, _vp, _vp],
    "ffca_transform": [_i, _vp, _i, _i, _i, _i, _i, _i, _vp, _vp, _vp],
    "ffca_mixture_weights": [_i, _vp, _i, _i, _i, _i, _i, _i, _i, _vp, _vp, _vp],
    "ffca_fastfca_estep_yt": [_i, _vp, _i, _i, _i, _i, _i, _i, _i, _vp, _vp, _vp, _vp, _vp],
    "ffca_fca_mstep": [_i, _vp, _i, _i, _i, _i, _i, _i, _i, _vp, _vp, _vp, _i, _d, _vp, _vp, _vp, _vp],
    "ffca_power_floor": [_i, _vp, _i, _i, _i, _i, _i, _i, _vp, _vp],
    "ffca_reconstruct_covariances": [_i, _vp, _i, _i, _i, _i, _i, _i, _vp, _vp, _vp, _vp],
    "ffca_back_transform_phi": [_i, _vp, _i, _i, _i, _i, _i, _i, _i, _vp, _vp, _vp, _vp],
    "ffca_params_from_covariances": [_i, _vp, _i, _i, _i, _i, _i, _i, _vp, _vp, _vp, _vp],
    "ffca_init_covariances": [_i, _vp, _i, _i, _i, _i, _i, _i, _i, _i, _vp, _vp, _vp, _vp, _vp],
    "ffca_sdr_energies": [_i, _vp, _i, _i, _i, _i, ctypes.c_longlong, ctypes.c_longlong, _vp, _vp, _vp],
    "ffca_stft_analyze": [_i, _vp, _i, _i, _i, ctypes.c_longlong, _i, _i, _vp, _vp],
    "ffca_stft_synthesize": [_i, _vp, _i, _i, _i, _i, _i, _i, _vp, _vp],
    "ffca_mstep_diag": [_i, _vp, _i, _i, _i, _i, _i, _i, _i, _vp, _vp, _vp, _i, _d, _vp, _vp, _vp],
}
_RESTYPES = {"ffca_last_error": ctypes.c_char_p, "ffca_set_kernel_timing": None,
             "ffca_last_kernel_ms": ctypes.c_float}

_lib = None
_device = int(os.environ.get("FFCA_DEVICE", "0"))


def load():
    """Load the CUDA library (once).  Raises BackendUnavailable if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise BackendUnavailable(
            f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, argtypes in SIGNATURES.items():
        fn = getattr(lib, name, None)
        if fn is None:  # reported by tests/test_abi_symbols.py
            continue
        fn.argtypes = argtypes
        fn.restype = _RESTYPES.get(name, ctypes.c_int)
    _lib = lib
    return lib


def set_device(device: int) -> None:
    global _device
    _device = int(device)


def device() -> int:
    return _device


def require_gpu():
    lib = load()
    if lib.ffca_device_count() < 1:
        raise BackendUnavailable("no CUDA device visible; the FastFCA-AS B200 path has no CPU fallback")
    return lib


def last_error() -> str:
    return (load().ffca_last_error() or b"").decode(errors="replace")


def check(rc: int, what: str = "") -> None:
    """Map an FFCA_E_* code onto the reference's exception types (errors.py)."""
    if rc == OK:
        return
    msg = f"{what}: {last_error()}" if what else last_error()
    if rc == E_SINGULAR_P:
        raise SingularP(msg)
    if rc == E_SINGULAR_B:
        raise SingularWeightedCovariance(msg)
    if rc == E_NOT_PD:
        raise NotPositiveDefinite(msg)
    if rc == E_ARG:
        raise DimensionMismatch(msg)
    if rc == E_UNSUPPORTED:
        raise DimensionMismatch(msg)
    raise RuntimeError(f"CUDA failure in {what}: {last_error()}")


def ptr(a) -> int | None:
    """Data pointer of a C-contiguous numpy array (or None)."""
    if a is None:
        return None
    if not a.flags["C_CONTIGUOUS"]:
        raise ValueError("array must be C-contiguous")
    return a.ctypes.data


def dtype_code(arr_dtype) -> int:
    return C64 if np.dtype(arr_dtype) in (np.dtype(np.complex64), np.dtype(np.float32)) else C128


def real_dtype(code: int):
    return np.float32 if code == C64 else np.float64


def complex_dtype(code: int):
    return np.complex64 if code == C64 else np.complex128


def launches() -> int:
    return int(load().ffca_last_launch_count())

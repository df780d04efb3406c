"""ctypes binding of libecc_b200.so (the C ABI in include/ecc_b200.h).

There is no CPU fallback: if the library or a CUDA device is missing every
entry point raises.  Device buffers are torch tensors; streams are torch's
current CUDA stream.
"""

from __future__ import annotations

import ctypes
import os
from contextlib import contextmanager
from pathlib import Path

import numpy as np
import torch

# ECC_B200_LIB: an alternative in-tree build (kernel A/B experiments under tools/)
_LIB_PATH = Path(os.environ.get("ECC_B200_LIB") or Path(__file__).resolve().parent / "libecc_b200.so")
_lib = None

ECC_OK = 0
ECC_EINVAL = -22
ECC_ECUDA = -5
DTYPE_U8, DTYPE_F32, DTYPE_F64 = 0, 1, 2

_TORCH_DTYPE = {torch.uint8: DTYPE_U8, torch.float32: DTYPE_F32, torch.float64: DTYPE_F64}


class EngineUnavailable(RuntimeError):
    """The CUDA engine cannot run here (library not built or no GPU)."""


class Binning(ctypes.Structure):
    _fields_ = [("t0", ctypes.c_double), ("inv_w", ctypes.c_double), ("nbins", ctypes.c_int64),
                ("mode", ctypes.c_int32), ("max_correction", ctypes.c_int32), ("lut_scale", ctypes.c_float),
                ("lut_bias", ctypes.c_float), ("lut_cells", ctypes.c_int32), ("lut_ok", ctypes.c_int32),
                ("lut_edge", ctypes.c_int32), ("lut_edge_sub", ctypes.c_int32)]


class SoftParams(ctypes.Structure):
    _fields_ = [("lam", ctypes.c_double), ("alpha", ctypes.c_double), ("u", ctypes.c_double * 3),
                ("center", ctypes.c_double), ("factorized", ctypes.c_int32), ("pad", ctypes.c_int32)]


def lib():
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            raise EngineUnavailable(
                f"{_LIB_PATH} is missing; build it with `python -m paper_2510_20271_b200.build`")
        L = ctypes.CDLL(str(_LIB_PATH))
        vp, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
        L.ecc_version.restype = ctypes.c_char_p
        L.ecc_last_error.restype = ctypes.c_char_p
        L.ecc_threshold_table.argtypes = [vp, i64, i32, vp, ctypes.POINTER(Binning)]
        L.ecc_threshold_table_bytes.argtypes = [i64, i32]
        L.ecc_threshold_table_bytes.restype = ctypes.c_size_t
        L.ecc_histogram.argtypes = [vp, i32, i32, vp, i64, vp, ctypes.POINTER(Binning), vp, vp]
        L.ecc_histogram_range.argtypes = [vp, i32, i32, vp, i64, i64, i64, vp, ctypes.POINTER(Binning), vp, vp]
        if hasattr(L, "ecc_histogram_checked"):   # absent from older builds used in A/B tools
            L.ecc_histogram_checked.argtypes = [vp, i32, i32, vp, i64, i64, i64, vp, ctypes.POINTER(Binning), vp,
                                                vp, vp]
        L.ecc_scan.argtypes = [vp, i64, i64, vp, vp]
        L.ecc_coefficients.argtypes = [vp, i32, i32, vp, i64, vp, vp]
        L.ecc_minmax.argtypes = [vp, i32, i64, vp, vp]
        L.ecc_key_to_double.argtypes = [ctypes.c_uint64]
        L.ecc_key_to_double.restype = ctypes.c_double
        L.ecc_soft_workspace_bytes.argtypes = [i32, vp, i64, i64]
        L.ecc_soft_workspace_bytes.restype = ctypes.c_size_t
        L.ecc_soft_prepare.argtypes = [vp, i32, i32, vp, i64, ctypes.POINTER(SoftParams), vp, vp, vp, vp]
        L.ecc_soft_forward.argtypes = [vp, vp, vp, i32, vp, i64, vp, i64, ctypes.POINTER(SoftParams), vp, vp, vp]
        L.ecc_soft_backward.argtypes = [vp, vp, vp, i32, vp, i64, vp, i64, ctypes.POINTER(SoftParams), vp, vp,
                                        vp, vp, vp, vp]
        L.ecc_effective_field.argtypes = [vp, i32, i32, vp, i64, ctypes.c_double, vp, vp, vp]
        L.ecc_counter_grid.argtypes = [ctypes.c_uint64, i64, i64, vp, vp]
        dbl = ctypes.c_double
        L.ecc_soft_fd.argtypes = [vp, vp, i32, vp, vp, i64, vp, dbl, dbl, vp, dbl, vp, vp, vp, vp]
        if hasattr(L, "ecc_soft_setup"):
            L.ecc_soft_setup.argtypes = [vp, i64, vp, i32, vp, dbl, vp, vp]
            L.ecc_soft_prepare_d.argtypes = [vp, i32, i32, vp, i64, vp, vp, vp, vp, vp]
            L.ecc_soft_forward_d.argtypes = [vp, vp, vp, i32, vp, i64, vp, i64, vp, vp, vp, vp, vp]
            L.ecc_soft_backward_d.argtypes = [vp, vp, vp, i32, vp, i64, vp, i64, vp, vp, vp, vp, vp, vp, vp, vp]
        if hasattr(L, "ecc_soft_records_bytes"):
            L.ecc_soft_records_bytes.argtypes = [i32, vp, i64]
            L.ecc_soft_records_bytes.restype = ctypes.c_size_t
        if hasattr(L, "ecc_soft_forward_range_d"):
            L.ecc_soft_prepare_range_d.argtypes = [vp, i32, i32, vp, i64, vp, vp, vp, vp, i64, i64, vp]
            L.ecc_soft_units.argtypes = [i32, vp, i64, vp, vp]
            L.ecc_soft_forward_range_d.argtypes = [vp, vp, vp, i32, vp, i64, vp, i64, vp, vp, vp, vp, i64, i64, i64,
                                                   i64, i64, i32, vp]
            L.ecc_soft_backward_range_d.argtypes = [vp, vp, vp, i32, vp, i64, vp, i64, vp, vp, vp, vp, vp, vp, vp,
                                                    i64, i64, i64, i64, i64, i32, vp]
        _lib = L
        if hasattr(L, "ecc_set_variant"):
            L.ecc_set_variant.argtypes = [ctypes.c_char_p, ctypes.c_char_p]
            _apply_env_variants()
    return _lib


# Kernel-variant switches (A/B checks; ecc_set_variant in the C ABI).  The
# launchers never read the environment; for the development tools the legacy
# ECC_B200_* variables are applied once, when the library is loaded.
_VARIANT_DEFAULTS = {"f3": "default", "zunit": "0", "generic": "0", "soft_fwd_t": "16", "soft_bwd_t": "16",
                     "soft_band": "1", "soft_g": "0", "soft_prep": "0"}
_VARIANT_ENV = {"f3": "ECC_B200_F3", "zunit": "ECC_B200_F3_ZUNIT", "generic": "ECC_B200_GENERIC",
                "soft_fwd_t": "ECC_SOFT_FWD_T", "soft_bwd_t": "ECC_SOFT_BWD_T",
                "soft_band": "ECC_SOFT_BAND", "soft_g": "ECC_SOFT_G",
                "soft_prep": "ECC_SOFT_PREP"}


def set_variant(key: str, value) -> None:
    check(lib().ecc_set_variant(key.encode(), str(value).encode()))


def _apply_env_variants() -> None:
    for key, env in _VARIANT_ENV.items():
        v = os.environ.get(env)
        if v:
            set_variant(key, v)


@contextmanager
def variant(**kw):
    """Run a block with kernel variants switched (f3=..., zunit=..., generic=1,
    soft_fwd_t=..., soft_bwd_t=..., soft_band=0/1, soft_g=chunks per CTA, soft_prep=1 (old 3-D prepare)); the production defaults are restored after."""
    for k, v in kw.items():
        set_variant(k, v)
    try:
        yield
    finally:
        for k in kw:
            set_variant(k, _VARIANT_DEFAULTS[k])


def check(rc: int):
    if rc == ECC_OK:
        return
    msg = lib().ecc_last_error().decode(errors="replace")
    if rc == ECC_EINVAL:
        raise ValueError(msg)
    raise RuntimeError(f"ecc_b200 CUDA failure ({rc}): {msg}")


def device() -> torch.device:
    """The CUDA device the engine runs on; raises when there is none."""
    if not torch.cuda.is_available():
        raise EngineUnavailable("ecc_b200 needs a CUDA device (sm_100a); none is visible")
    lib()
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr(t: torch.Tensor | None = None) -> ctypes.c_void_p:
    dev = t.device if t is not None else None
    return ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def ptr(t: torch.Tensor | np.ndarray | None) -> ctypes.c_void_p:
    if t is None:
        return ctypes.c_void_p(0)
    if isinstance(t, np.ndarray):
        return t.ctypes.data_as(ctypes.c_void_p)
    return ctypes.c_void_p(t.data_ptr())


def dims_arg(shape) -> np.ndarray:
    return np.ascontiguousarray(np.array(list(shape), dtype=np.int64))


def dtype_code(t: torch.Tensor) -> int:
    try:
        return _TORCH_DTYPE[t.dtype]
    except KeyError:
        raise ValueError(f"unsupported grid dtype {t.dtype}; expected uint8, float32 or float64") from None


def version() -> str:
    return lib().ecc_version().decode()

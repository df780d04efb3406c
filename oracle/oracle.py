"""CPU oracle for the ECC hot paths -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this module.  The product package
(paper_2510_20271_b200) never does; if its CUDA library is missing it fails
loudly instead of falling back here.

This is a ctypes wrapper over oracle/ecc_oracle.c, a plain-C restatement of
the reference (ecckit 0.1.0, /root/reference/pkg/src/ecckit):

* coefficients  -- coefficients.py:74-138  (_lower_masks/_lower_star_coefficients)
* histogram     -- hard.py:121-143, 184-212 (packed bincount + fold == per-bin sum of c)
* binning       -- grid.py:168-180 (searchsorted side='left' over float64 taus)
* curve         -- hard.py:215-226 (cumsum)
* soft forward  -- soft.py:154-196
* soft backward -- soft.py:199-257 (+ G = sum c w pos for d_alpha)
* effective field -- soft.py:79-101 with OpenBLAS's dgemv FMA order

Parity is pinned: tests/test_oracle_golden.py checks every function against
tests/golden/golden.npz, produced by running the reference itself
(tests/golden/make_golden.py).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "_build" / "libecc_oracle.so"
_lib = None

_i64p = ctypes.POINTER(ctypes.c_int64)
_f64p = ctypes.POINTER(ctypes.c_double)


def build() -> Path:
    """Compile the C oracle (make)."""
    subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            build()
        L = ctypes.CDLL(str(_LIB_PATH))
        vp = ctypes.c_void_p
        L.ecc_oracle_coefficients.argtypes = [vp, ctypes.c_int, vp, vp]
        L.ecc_oracle_histogram.argtypes = [vp, ctypes.c_int, vp, vp, ctypes.c_int64, vp]
        L.ecc_oracle_histogram_rows.argtypes = [vp, ctypes.c_int, vp, ctypes.c_int64, ctypes.c_int64, vp,
                                                ctypes.c_int64, vp]
        L.ecc_oracle_histogram_f32.argtypes = [vp, ctypes.c_int, vp, vp, ctypes.c_int64, vp]
        L.ecc_oracle_histogram_rows_f32.argtypes = [vp, ctypes.c_int, vp, ctypes.c_int64, ctypes.c_int64, vp,
                                                    ctypes.c_int64, vp]
        L.ecc_oracle_curve.argtypes = [vp, ctypes.c_int, vp, vp, ctypes.c_int64, vp]
        L.ecc_oracle_effective_field.argtypes = [vp, ctypes.c_int, vp, ctypes.c_double, vp, vp]
        L.ecc_oracle_soft_forward.argtypes = [vp, vp, ctypes.c_int, vp, ctypes.c_double, ctypes.c_double, vp, vp,
                                              ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, vp]
        L.ecc_oracle_soft_backward.argtypes = [vp, vp, ctypes.c_int, vp, ctypes.c_double, ctypes.c_double, vp, vp,
                                               ctypes.c_int64, vp, vp, vp, vp]
        L.ecc_oracle_counter_grid.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64, vp]
        L.ecc_oracle_num_threads.restype = ctypes.c_int
        L.ecc_oracle_set_threads.argtypes = [ctypes.c_int]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _dims(x: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(np.array(x.shape, dtype=np.int64))


def num_threads() -> int:
    return int(lib().ecc_oracle_num_threads())


def set_threads(n: int) -> None:
    """Thread count of the parallel loops (the reference's ``workers``)."""
    lib().ecc_oracle_set_threads(int(n))


def coefficients(values) -> np.ndarray:
    x = np.ascontiguousarray(values, dtype=np.float64)
    out = np.empty(x.shape, dtype=np.int8)
    d = _dims(x)
    lib().ecc_oracle_coefficients(_p(x), x.ndim, _p(d), _p(out))
    return out


def histogram(values, taus) -> tuple[np.ndarray, int]:
    """(bins[B] int64, overflow int) -- HistogramBins.bins / .overflow."""
    taus = np.ascontiguousarray(taus, dtype=np.float64)
    out = np.zeros(taus.size + 1, dtype=np.int64)
    v = np.asarray(values)
    if v.dtype == np.float32:
        x = np.ascontiguousarray(v)
        d = _dims(x)
        lib().ecc_oracle_histogram_f32(_p(x), x.ndim, _p(d), _p(taus), taus.size, _p(out))
    else:
        x = np.ascontiguousarray(v, dtype=np.float64)
        d = _dims(x)
        lib().ecc_oracle_histogram(_p(x), x.ndim, _p(d), _p(taus), taus.size, _p(out))
    return out[:-1].copy(), int(out[-1])


def histogram_rows(values, r0: int, r1: int, taus) -> np.ndarray:
    """bins+overflow (B+1) of axis-0 rows [r0, r1) of a slab with halo rows."""
    taus = np.ascontiguousarray(taus, dtype=np.float64)
    out = np.zeros(taus.size + 1, dtype=np.int64)
    v = np.asarray(values)
    if v.dtype == np.float32:
        x = np.ascontiguousarray(v)
        d = _dims(x)
        lib().ecc_oracle_histogram_rows_f32(_p(x), x.ndim, _p(d), r0, r1, _p(taus), taus.size, _p(out))
    else:
        x = np.ascontiguousarray(v, dtype=np.float64)
        d = _dims(x)
        lib().ecc_oracle_histogram_rows(_p(x), x.ndim, _p(d), r0, r1, _p(taus), taus.size, _p(out))
    return out


def curve(values, taus) -> np.ndarray:
    bins, _ = histogram(values, taus)
    return np.cumsum(bins)


def effective_field(values, alpha: float, u) -> np.ndarray:
    x = np.ascontiguousarray(values, dtype=np.float64)
    u = np.ascontiguousarray(np.asarray(u, dtype=np.float64).ravel())
    out = np.empty_like(x)
    d = _dims(x)
    lib().ecc_oracle_effective_field(_p(x), x.ndim, _p(d), float(alpha), _p(u), _p(out))
    return out


def soft_forward(values, coeffs, lam, alpha, u, taus, p0: int = 0, p1: int | None = None) -> np.ndarray:
    x = np.ascontiguousarray(values, dtype=np.float64)
    c = np.ascontiguousarray(coeffs, dtype=np.int8)
    u = np.ascontiguousarray(np.asarray(u, dtype=np.float64).ravel())
    taus = np.ascontiguousarray(taus, dtype=np.float64)
    chi = np.empty(taus.size)
    d = _dims(x)
    p1 = x.size if p1 is None else p1
    lib().ecc_oracle_soft_forward(_p(x), _p(c), x.ndim, _p(d), float(lam), float(alpha), _p(u), _p(taus),
                                  taus.size, int(p0), int(p1), _p(chi))
    return chi


def soft_backward(values, coeffs, lam, alpha, u, taus, upstream):
    """Returns (d_values, d_tau, d_u_projected, d_alpha, G) -- soft.py:199-257."""
    x = np.ascontiguousarray(values, dtype=np.float64)
    c = np.ascontiguousarray(coeffs, dtype=np.int8)
    u = np.ascontiguousarray(np.asarray(u, dtype=np.float64).ravel())
    taus = np.ascontiguousarray(taus, dtype=np.float64)
    up = np.ascontiguousarray(upstream, dtype=np.float64)
    dv = np.empty(x.shape)
    dt = np.empty(taus.size)
    G = np.zeros(3)
    d = _dims(x)
    lib().ecc_oracle_soft_backward(_p(x), _p(c), x.ndim, _p(d), float(lam), float(alpha), _p(u), _p(taus),
                                   taus.size, _p(up), _p(dv), _p(dt), _p(G))
    G = G[: x.ndim]
    du = -alpha * G
    du = du - (du @ u) * u
    dalpha = -float(G @ u)
    return dv, dt, du, dalpha, G


def counter_grid(seed: int, dims, start: int = 0, count: int | None = None) -> np.ndarray:
    n = int(np.prod(dims))
    count = n - start if count is None else count
    out = np.empty(count, dtype=np.float32)
    lib().ecc_oracle_counter_grid(ctypes.c_uint64(seed), start, count, _p(out))
    return out

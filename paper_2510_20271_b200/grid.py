"""Grid model, threshold sets and curves -- the types of ecckit/grid.py.

Mirrors the reference's public types (grid.py:39-228) so callers can switch
imports.  The difference is where the data lives: a ScalarGrid keeps a
device copy in the narrowest dtype that represents its values exactly
(uint8, float32 or float64), which is what the CUDA kernels read.  The
float64 host view (`.values`) that the reference exposes is materialised
lazily.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib


class FormatError(ValueError):
    """File does not conform to the grid file format (grid.py:39-40)."""


class CorruptionError(ValueError):
    """Structurally valid header whose payload does not match it (grid.py:43-44)."""


def _narrowest_exact(arr64: np.ndarray) -> np.ndarray:
    """uint8 / float32 / float64 array with identical values under comparison
    (grid.py:5-8: files and generators produce float32-representable grids)."""
    a32 = arr64.astype(np.float32)
    if not np.array_equal(a32.astype(np.float64), arr64):
        return arr64
    if arr64.size and arr64.min() >= 0 and arr64.max() <= 255 and np.array_equal(np.floor(arr64), arr64):
        return arr64.astype(np.uint8)
    return a32


class ScalarGrid:
    """An immutable dense 2D/3D scalar field (grid.py:47-81).

    ``values`` may be array-like (copied, validated on the host exactly like
    the reference) or a CUDA tensor (kept on device, validated there).
    """

    def __init__(self, values):
        if isinstance(values, ScalarGrid):
            self._dev, self._host = values._dev, values._host
            return
        if isinstance(values, torch.Tensor) and values.is_cuda:
            t = values.detach()
            if t.ndim not in (2, 3):
                raise ValueError(f"grid must be 2D or 3D, got ndim={t.ndim}")
            if any(s < 1 for s in t.shape):
                raise ValueError(f"grid extents must be positive, got {tuple(t.shape)}")
            if t.dtype not in (torch.uint8, torch.float32, torch.float64):
                t = t.to(torch.float64)
            t = t.contiguous()
            if t.dtype != torch.uint8:
                from .hard import device_minmax
                _, _, bad = device_minmax(t)
                if bad:
                    raise ValueError("grid values must be finite (no NaN/Inf)")
            self._dev = t
            self._host = None
            return
        arr = np.array(values.cpu().numpy() if isinstance(values, torch.Tensor) else values,
                       dtype=np.float64, order="C")
        if arr.ndim not in (2, 3):
            raise ValueError(f"grid must be 2D or 3D, got ndim={arr.ndim}")
        if any(s < 1 for s in arr.shape):
            raise ValueError(f"grid extents must be positive, got {arr.shape}")
        if not np.isfinite(arr).all():
            raise ValueError("grid values must be finite (no NaN/Inf)")
        arr.flags.writeable = False
        self._host = arr
        self._dev = None

    # -- reference surface ---------------------------------------------------
    @property
    def values(self) -> np.ndarray:
        if self._host is None:
            arr = self._dev.to(torch.float64).cpu().numpy()
            arr.flags.writeable = False
            self._host = arr
        return self._host

    @property
    def dims(self) -> tuple[int, ...]:
        return tuple(self._dev.shape) if self._dev is not None else self._host.shape

    @property
    def ndim(self) -> int:
        return len(self.dims)

    @property
    def size(self) -> int:
        n = 1
        for d in self.dims:
            n *= d
        return n

    def __repr__(self):
        return f"ScalarGrid(dims={self.dims})"

    # -- engine surface --------------------------------------------------------
    def device_tensor(self) -> torch.Tensor:
        """Contiguous CUDA tensor (uint8/float32/float64) holding the values exactly."""
        if self._dev is None:
            dev = _lib.device()
            self._dev = torch.from_numpy(np.array(_narrowest_exact(self._host), order="C", copy=True)).to(dev)
        return self._dev


def flatten_index(coords, dims) -> int:
    """Row-major linear index of a pixel coordinate tuple (grid.py:84-86)."""
    return int(np.ravel_multi_index(tuple(coords), tuple(dims)))


def unflatten_index(index: int, dims) -> tuple[int, ...]:
    """Inverse of :func:`flatten_index` (grid.py:89-93)."""
    if index < 0:
        raise ValueError(f"negative linear index {index}")
    return tuple(int(c) for c in np.unravel_index(index, tuple(dims)))


class ThresholdSet:
    """Strictly increasing, finite thresholds (grid.py:115-180).

    Validation is the reference's.  Binning on the device uses per-dtype
    compare tables (float32 round-down copies for float32/uint8 grids, the
    float64 values for float64 grids) built by ecc_threshold_table, which
    also certifies the affine guess (grid.py:147-166) or selects binary
    search; both are exact.
    """

    def __init__(self, taus):
        arr = np.array(taus, dtype=np.float64).ravel()
        if arr.size < 1:
            raise ValueError("threshold set must contain at least one value")
        if not np.isfinite(arr).all():
            raise ValueError("thresholds must be finite")
        if arr.size > 1 and not (np.diff(arr) > 0).all():
            raise ValueError("thresholds must be strictly increasing")
        arr.flags.writeable = False
        self.taus = arr
        self._tables: dict = {}

    def __len__(self) -> int:
        return self.taus.size

    def __repr__(self):
        return f"ThresholdSet(n={len(self)}, lo={self.taus[0]}, hi={self.taus[-1]})"

    def bin_indices(self, values) -> np.ndarray:
        """Smallest j with value <= taus[j]; len(self) above the last (grid.py:168-180).

        Host utility for API compatibility (binary search); the engine bins on
        the device inside the fused sweep.
        """
        return np.searchsorted(self.taus, np.asarray(values, dtype=np.float64), side="left")

    def device_table(self, dtype_code: int, device: torch.device):
        """(table tensor on device, Binning struct) for a grid dtype."""
        key = (dtype_code, str(device))
        hit = self._tables.get(key)
        if hit is None:
            nb = self.taus.size
            nbytes = int(_lib.lib().ecc_threshold_table_bytes(nb, dtype_code))
            host = np.zeros(nbytes // 4 + 1, dtype=np.float32)
            if dtype_code == _lib.DTYPE_F64:
                host = np.zeros(nbytes // 8 + 1, dtype=np.float64)
            b = _lib.Binning()
            taus = np.ascontiguousarray(self.taus)
            _lib.check(_lib.lib().ecc_threshold_table(_lib.ptr(taus), nb, dtype_code, _lib.ptr(host),
                                                      _lib.ctypes.byref(b)))
            hit = (torch.from_numpy(host).to(device), b, host)
            self._tables[key] = hit
        return hit[0], hit[1]


def uniform_thresholds(grid: ScalarGrid, bins: int) -> ThresholdSet:
    """Right edges of `bins` equal-width intervals over [min, max] (grid.py:183-196).

    min/max come from the device (ecc_minmax); the edge formula is the
    reference's, in float64 on the host.
    """
    if bins < 1:
        raise ValueError(f"bins must be >= 1, got {bins}")
    from .hard import device_minmax
    lo, hi, _ = device_minmax(grid.device_tensor())
    return thresholds_from_range(lo, hi, bins)


def thresholds_from_range(lo: float, hi: float, bins: int) -> ThresholdSet:
    edges = lo + (hi - lo) * (np.arange(1, bins + 1) / bins)
    edges[-1] = hi
    return ThresholdSet(np.unique(edges))


class EulerCurve:
    """Threshold/value pairs of an Euler characteristic curve (grid.py:199-228)."""

    def __init__(self, taus, values):
        taus = np.asarray(taus, dtype=np.float64)
        values = np.asarray(values)
        if values.dtype.kind not in "if":
            raise ValueError(f"curve values must be numeric, got {values.dtype}")
        if taus.shape != values.shape or taus.ndim != 1:
            raise ValueError(
                f"taus and values must be equal-length 1D arrays, "
                f"got {taus.shape} and {values.shape}"
            )
        self.taus = taus
        self.values = values

    @property
    def is_integral(self) -> bool:
        return self.values.dtype.kind == "i"

    def __len__(self) -> int:
        return self.taus.size

    def __repr__(self):
        kind = "int" if self.is_integral else "float"
        return f"EulerCurve(n={len(self)}, {kind})"

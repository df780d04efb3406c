"""Per-voxel Euler characteristic coefficients (ecckit/coefficients.py) on the GPU.

c(p) = 1 - e(p) + f(p) - b(p) over the cells p owns under the (value,
linear index) order (coefficients.py:1-25); computed by the same stencil
code the fused histogram sweep uses (csrc/ecc_common.cuh coeff3).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .grid import ScalarGrid

#: Inclusive attainable coefficient ranges by grid dimension (coefficients.py:44).
COEFF_RANGE = {2: (-3, 1), 3: (-5, 7)}


@dataclass(frozen=True)
class CoefficientGrid:
    """Integer coefficients, one per pixel of the source grid (coefficients.py:47-63)."""

    coeffs: np.ndarray

    def __post_init__(self):
        if self.coeffs.ndim not in (2, 3):
            raise ValueError(f"coefficients must be 2D or 3D, got {self.coeffs.ndim}")

    @property
    def dims(self) -> tuple[int, ...]:
        return self.coeffs.shape

    @property
    def ndim(self) -> int:
        return self.coeffs.ndim


def coefficients_device(x: torch.Tensor, ndim: int | None = None) -> torch.Tensor:
    """int8 coefficients of CUDA grids x [N?, (D,) H, W]."""
    from .hard import _split_batch

    x = x.contiguous()
    batch, dims, _ = _split_batch(x, ndim)
    out = torch.empty(x.shape, dtype=torch.int8, device=x.device)
    d = _lib.dims_arg(dims)
    _lib.check(_lib.lib().ecc_coefficients(_lib.ptr(x), _lib.dtype_code(x), len(dims), _lib.ptr(d), batch,
                                           _lib.ptr(out), _lib.stream_ptr(x)))
    return out


def compute_coefficients(grid: ScalarGrid) -> CoefficientGrid:
    """Euler characteristic coefficients of every pixel (coefficients.py:163-175)."""
    c = coefficients_device(grid.device_tensor())
    return CoefficientGrid(c.cpu().numpy())


def vertex_order(grid: ScalarGrid) -> np.ndarray:
    """Permutation sorting pixels by (value, index) (coefficients.py:178-180)."""
    t = grid.device_tensor().reshape(-1)
    if t.dtype == torch.uint8:
        t = t.to(torch.int16)
    return torch.sort(t, stable=True).indices.cpu().numpy()

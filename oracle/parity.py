"""Oracle results for the benchmarked configurations -- TEST INFRASTRUCTURE ONLY.

The GPU parity tests (tests/test_gpu_timed.py) and bench.py's per-leg gate
compute the reference answer of exactly the volume they time with these
helpers; the product package never imports them.

* ``counter_slab_hist`` -- the int64 histogram (B bins + overflow) of planes
  [z0, z1) of the counter-generated volume (splitmix64 of the
  linear index, ecc_oracle.c), accumulated slab by slab through
  ``oracle.histogram_rows`` (the reference's row blocks with a one-row halo,
  coefficients.py:141-152, merged as hard.py:99-118), so 1024^3 and the C5
  slab never materialise on the host.
* ``soft_item`` -- forward chi and the backward gradients of one soft item
  (soft.py:154-257, plus d_alpha).
"""

from __future__ import annotations

import numpy as np

from . import oracle


def counter_slab_hist(seed: int, dims, z0: int, z1: int, taus, slab: int = 64) -> np.ndarray:
    """B+1 int64 histogram of planes [z0, z1) of the counter volume `dims` (D, H, W)."""
    D, H, W = (int(d) for d in dims)
    plane = H * W
    taus = np.ascontiguousarray(taus, dtype=np.float64)
    out = np.zeros(taus.size + 1, dtype=np.int64)
    for a in range(z0, z1, slab):
        b = min(a + slab, z1)
        lo, hi = max(a - 1, 0), min(b + 1, D)          # halo planes where they exist
        x = oracle.counter_grid(seed, (D, H, W), start=lo * plane, count=(hi - lo) * plane)
        x = x.reshape(hi - lo, H, W)
        out += oracle.histogram_rows(x, a - lo, b - lo, taus)
    return out


def soft_item(x, lam: float, alpha: float, u, taus, upstream):
    """(chi, d_values, d_tau, d_u_projected, d_alpha, G) of one grid x (float64),
    coefficients of the effective field frozen as in the reference tests
    (test_soft.py:220-222)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    c = oracle.coefficients(oracle.effective_field(x, alpha, u))
    chi = oracle.soft_forward(x, c, lam, alpha, u, taus)
    dv, dt, du, da, G = oracle.soft_backward(x, c, lam, alpha, u, taus, upstream)
    return chi, dv, dt, du, da, G

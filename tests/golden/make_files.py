"""Generate golden FILES (.eccg grids/coefficients, curve CSVs) by running the
REFERENCE (ecckit) in this container; run once, here:

    python tests/golden/make_files.py

The files are committed under tests/golden/files/ and pin the file formats of
grid.py:11-21 / coefficients.py:183-197 / grid.py:300-323 byte for byte.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from ecckit import (  # noqa: E402
    ScalarGrid,
    SyntheticSpec,
    generate_grid,
    SoftEccParams,
    compute_coefficients,
    compute_ecc,
    effective_field,
    reparametrize_direction,
    soft_ecc,
    uniform_thresholds,
    write_coefficients,
    write_curve,
    write_grid,
)

OUT = Path(__file__).resolve().parent / "files"


def main():
    OUT.mkdir(exist_ok=True)
    rng = np.random.default_rng(20261018)
    g2 = ScalarGrid(rng.random((13, 17)).astype(np.float32).astype(np.float64))
    g3 = ScalarGrid(rng.random((9, 11, 12)).astype(np.float32).astype(np.float64))
    write_grid(g2, OUT / "g2d.eccg")
    write_grid(g3, OUT / "g3d.eccg")
    write_coefficients(compute_coefficients(g3), OUT / "c3d.eccg")
    write_curve(compute_ecc(g3, uniform_thresholds(g3, 32)), OUT / "curve_g3d_32.csv")
    u = reparametrize_direction([1.0, 2.0])
    f = effective_field(g2, 0.3, u)
    ts = uniform_thresholds(f, 16)
    params = SoftEccParams(lam=50.0, alpha=0.3, u=u, taus=ts)
    write_curve(soft_ecc(g2, compute_coefficients(f), params), OUT / "soft_g2d_16.csv")
    write_grid(generate_grid(SyntheticSpec(kind="gaussian-blobs", dims=(12, 10), seed=4, blobs=3)),
               OUT / "blobs_12x10_s4_b3.eccg")
    write_grid(generate_grid(SyntheticSpec(kind="radial-gradient", dims=(5, 6, 7))), OUT / "radial_5x6x7.eccg")
    write_grid(generate_grid(SyntheticSpec(kind="uniform-random", dims=(4, 5, 6), seed=9)), OUT / "uniform_4x5x6_s9.eccg")
    for p in sorted(OUT.iterdir()):
        print(p.name, p.stat().st_size)


if __name__ == "__main__":
    main()

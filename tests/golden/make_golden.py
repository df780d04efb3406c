"""Generate golden vectors by running the REFERENCE (ecckit) in this container.

Run once, here (needs /root/reference; it does not exist on the GPU box):

    python tests/golden/make_golden.py

Writes tests/golden/golden.npz (committed).  Every array is produced by the
reference's own public functions (or, for d_alpha, by the reference's own
forward `_forward_raw` under the 4th-order stencil of soft.py:308-315), so
the tests that read this file pin both the CPU oracle (oracle/) and the CUDA
engine to the reference's outputs bit for bit (integer paths) or to a stated
tolerance (soft paths).
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from ecckit import (  # noqa: E402
    ScalarGrid,
    SoftEccParams,
    SyntheticSpec,
    ThresholdSet,
    accumulate_histogram,
    compute_coefficients,
    compute_ecc,
    effective_field,
    generate_grid,
    reparametrize_direction,
    soft_ecc,
    soft_ecc_backward,
    uniform_thresholds,
)
from ecckit.soft import _forward_raw  # noqa: E402

OUT = Path(__file__).with_name("golden.npz")


def main():
    rng = np.random.default_rng(20261018)
    arrays: dict[str, np.ndarray] = {}
    idx = {"coeff": 0, "hist": 0, "soft": 0, "uthr": 0}

    def add_coeff(vals):
        g = ScalarGrid(vals)
        k = idx["coeff"]
        arrays[f"coeff{k}_x"] = g.values
        arrays[f"coeff{k}_c"] = compute_coefficients(g).coeffs
        idx["coeff"] += 1

    def add_hist(vals, taus):
        g = ScalarGrid(vals)
        ts = taus if isinstance(taus, ThresholdSet) else ThresholdSet(taus)
        h = accumulate_histogram(g, ts)
        k = idx["hist"]
        arrays[f"hist{k}_x"] = g.values
        arrays[f"hist{k}_taus"] = ts.taus
        arrays[f"hist{k}_bins"] = h.bins
        arrays[f"hist{k}_overflow"] = np.array([h.overflow], dtype=np.int64)
        arrays[f"hist{k}_curve"] = compute_ecc(g, ts).values
        idx["hist"] += 1

    # --- coefficient fixtures (test_coefficients.py:29-69) -----------------
    add_coeff([[5.0]])
    add_coeff(np.zeros((2, 2)))
    add_coeff(np.zeros((2, 2, 2)))
    add_coeff(np.array([[9, 0, 9], [0, 5, 0], [9, 0, 9]], dtype=np.float64))
    v = np.full((3, 3, 3), 9.0)
    v[1, 1, 1] = 5.0
    for axis in range(3):
        for side in (0, 2):
            i = [1, 1, 1]
            i[axis] = side
            v[tuple(i)] = 0.0
    add_coeff(v.copy())
    for a in range(3):
        for b in range(a + 1, 3):
            for sa in (0, 2):
                for sb in (0, 2):
                    i = [1, 1, 1]
                    i[a], i[b] = sa, sb
                    v[tuple(i)] = 0.0
    add_coeff(v.copy())
    # random tie-heavy integer grids, f32 grids, +-0 / subnormal mixes
    for t in range(40):
        nd = 2 if t % 2 else 3
        dims = tuple(int(d) for d in rng.integers(1, 20 if nd == 2 else 8, nd))
        add_coeff(rng.integers(0, 4 if t % 3 else 10, dims).astype(np.float64))
    for t in range(20):
        nd = 2 if t % 2 else 3
        dims = tuple(int(d) for d in rng.integers(1, 24 if nd == 2 else 9, nd))
        add_coeff(rng.random(dims).astype(np.float32).astype(np.float64))
    specials = np.array([0.0, -0.0, 1e-45, -1e-45, 1.17549435e-38, -1.4e-45, 3.4e38, -3.4e38, 1.0, -1.0],
                        dtype=np.float32).astype(np.float64)
    for t in range(10):
        nd = 2 if t % 2 else 3
        dims = tuple(int(d) for d in rng.integers(2, 14 if nd == 2 else 7, nd))
        add_coeff(rng.choice(specials, size=dims))

    # --- histograms / curves (test_hard.py:27-50, test_grid.py:112-129) ------
    peak2 = np.zeros((3, 3))
    peak2[1, 1] = 1.0
    add_hist(peak2, [0.0, 1.0])
    peak3 = np.zeros((3, 3, 3))
    peak3[1, 1, 1] = 1.0
    add_hist(peak3, [0.0, 1.0])
    for t in range(30):
        nd = 2 if t % 2 else 3
        dims = tuple(int(d) for d in rng.integers(1, 40 if nd == 2 else 12, nd))
        vals = rng.integers(0, 10, dims).astype(np.float64)
        g = ScalarGrid(vals)
        taus = np.unique(vals) if t % 3 == 0 else uniform_thresholds(g, int(rng.integers(1, 40))).taus
        add_hist(vals, taus)
    for t in range(20):
        nd = 2 if t % 2 else 3
        dims = tuple(int(d) for d in rng.integers(1, 64 if nd == 2 else 20, nd))
        vals = rng.random(dims).astype(np.float32).astype(np.float64)
        g = ScalarGrid(vals)
        if t % 4 == 0:
            taus = np.sort(rng.normal(0.5, 0.3, int(rng.integers(1, 50))))
            taus = np.unique(taus)
        else:
            taus = uniform_thresholds(g, int(rng.integers(1, 300))).taus
        add_hist(vals, taus)
    # hostile threshold sets (test_grid.py:112-129) against f32 grids
    hostile = [
        np.array([1e15, 1e15 + 1, 1e15 + 2]),
        np.array([-1e300, 0.0, 1e300]),
        np.array([0.0, 1e-300, 2e-300, 1.0]),
        np.arange(64.0) * 1e-6 + 5e8,
        np.array([-1.0, -1e-45, 0.0, 1e-45, 0.5]),
    ]
    for taus in hostile:
        dims = (17, 13)
        vals = rng.choice(np.concatenate([taus, np.nextafter(taus, np.inf), np.nextafter(taus, -np.inf),
                                          rng.uniform(-2, 2, 10)]), size=dims)
        vals = np.clip(vals, -3.4e38, 3.4e38).astype(np.float32).astype(np.float64)
        add_hist(vals, taus)
    # C1 (BASELINE configs[0]): 2D 256x256 uint8, 256 uniform thresholds
    c1 = np.random.default_rng(1).integers(0, 256, (256, 256), np.uint8).astype(np.float64)
    add_hist(c1, uniform_thresholds(ScalarGrid(c1), 256))
    # a small uniform-random 3D volume through the reference generator
    g = generate_grid(SyntheticSpec("uniform-random", (48, 40, 36), seed=5))
    add_hist(g.values, uniform_thresholds(g, 1024))
    g = generate_grid(SyntheticSpec("gaussian-blobs", (32, 32, 32), seed=6))
    add_hist(g.values, uniform_thresholds(g, 128))

    # --- uniform_thresholds (grid.py:183-196) ------------------------------
    for t in range(20):
        dims = tuple(int(d) for d in rng.integers(1, 20, 2))
        vals = (rng.random(dims) * rng.uniform(1e-3, 1e3) - rng.uniform(-5, 5)).astype(np.float32).astype(np.float64)
        if t == 0:
            vals = np.full(dims, 4.25)
        bins = int(rng.integers(1, 300))
        k = idx["uthr"]
        arrays[f"uthr{k}_x"] = vals
        arrays[f"uthr{k}_bins"] = np.array([bins])
        arrays[f"uthr{k}_taus"] = uniform_thresholds(ScalarGrid(vals), bins).taus
        idx["uthr"] += 1

    # --- soft path (soft.py) ------------------------------------------------
    def add_soft(vals, alpha, u, lam, nb, upstream=None):
        g = ScalarGrid(vals)
        u = np.asarray(u, dtype=np.float64)
        eff = effective_field(g, alpha, u)
        taus = uniform_thresholds(eff, nb)
        coeffs = compute_coefficients(eff)
        params = SoftEccParams(lam=lam, alpha=alpha, u=u, taus=taus)
        if upstream is None:
            upstream = rng.uniform(0.5, 1.5, size=len(taus))
        chi = soft_ecc(g, coeffs, params).values
        grads = soft_ecc_backward(g, coeffs, params, upstream)
        step = 1e-4

        def loss_alpha(a):
            return float(upstream @ _forward_raw(g, coeffs, lam, a, u, taus))

        d_alpha = (-loss_alpha(alpha + 2 * step) + 8 * loss_alpha(alpha + step)
                   - 8 * loss_alpha(alpha - step) + loss_alpha(alpha - 2 * step)) / (12 * step)
        k = idx["soft"]
        arrays[f"soft{k}_x"] = g.values
        arrays[f"soft{k}_params"] = np.array([alpha, lam])
        arrays[f"soft{k}_u"] = u
        arrays[f"soft{k}_eff"] = eff.values
        arrays[f"soft{k}_taus"] = taus.taus
        arrays[f"soft{k}_coeffs"] = coeffs.coeffs
        arrays[f"soft{k}_upstream"] = np.asarray(upstream, dtype=np.float64)
        arrays[f"soft{k}_chi"] = chi
        arrays[f"soft{k}_dvalues"] = grads.d_values
        arrays[f"soft{k}_dtau"] = grads.d_tau
        arrays[f"soft{k}_du"] = grads.d_u
        arrays[f"soft{k}_dalpha_fd"] = np.array([d_alpha])
        idx["soft"] += 1

    add_soft(np.array([[0.0]]), 0.0, [1.0, 0.0], 4.0, 1, upstream=np.ones(1))
    for lam in (1.0, 10.0, 50.0):
        for alpha in (0.0, 0.3):
            vals = rng.integers(0, 10, (8, 8)) / 10.0
            add_soft(vals, alpha, reparametrize_direction(rng.normal(size=2)), lam, 6)
    add_soft(rng.integers(0, 10, (4, 4, 4)) / 10.0, 0.25, reparametrize_direction(rng.normal(size=3)), 10.0, 5)
    add_soft(rng.random((37, 23)).astype(np.float32).astype(np.float64), 0.3,
             reparametrize_direction([1.0, 2.0]), 50.0, 256)
    add_soft(rng.random((9, 8, 7)).astype(np.float32).astype(np.float64), 0.3,
             reparametrize_direction([1.0, 2.0, -0.5]), 50.0, 64)
    add_soft(rng.random((64, 64)).astype(np.float32).astype(np.float64), 0.3,
             reparametrize_direction([1.0, 2.0]), 50.0, 256)
    add_soft(rng.random((16, 16, 16)).astype(np.float32).astype(np.float64), 0.3,
             reparametrize_direction([1.0, 2.0, -0.5]), 50.0, 256)
    add_soft(rng.random((32, 32)), 0.2, reparametrize_direction([2.0, -1.0]), 8.0, 32)

    arrays["manifest"] = np.array([idx["coeff"], idx["hist"], idx["soft"], idx["uthr"]], dtype=np.int64)
    np.savez_compressed(OUT, **arrays)
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes): {idx}")


if __name__ == "__main__":
    main()

"""Shared test configuration.

Markers: ``gpu`` -- needs a CUDA device (run on the B200 box with
``pytest -m gpu``); everything else runs on the CPU-only build container.
The CPU oracle (oracle/) is imported here as the checker only.
"""

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = Path(__file__).resolve().parent / "golden" / "golden.npz"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def golden():
    return np.load(GOLDEN)


@pytest.fixture
def rng():
    return np.random.default_rng(20240817)


def golden_cases(g, prefix):
    n = dict(zip(["coeff", "hist", "soft", "uthr"], g["manifest"].tolist()))[prefix]
    return range(n)


def random_int_grid(rng, ndim, max_extent, lo=0, hi=9):
    """Random grid with integer-valued floats; plenty of ties (reference tests/conftest.py:9-12)."""
    dims = tuple(int(d) for d in rng.integers(1, max_extent + 1, ndim))
    return rng.integers(lo, hi + 1, dims).astype(np.float64)


def random_f32_grid(rng, ndim, max_extent):
    dims = tuple(int(d) for d in rng.integers(1, max_extent + 1, ndim))
    return rng.random(dims).astype(np.float32).astype(np.float64)


def normwise(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    den = max(np.abs(b).max(), 1e-300)
    return float(np.abs(a - b).max() / den)

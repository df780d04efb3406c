"""Grid / coefficient / curve files (ecckit grid.py:230-323, coefficients.py:183-197)
and the streaming loader.  The golden files in tests/golden/files were written
by the reference itself (tests/golden/make_files.py)."""

from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest
import torch

import paper_2510_20271_b200 as E
from oracle import oracle

FILES = Path(__file__).resolve().parent / "golden" / "files"


def _blob(path):
    return bytearray(Path(path).read_bytes())


class TestGoldenFiles:
    def test_grid_files_round_trip_byte_exact(self, tmp_path):
        for name in ("g2d.eccg", "g3d.eccg"):
            g = E.read_grid(FILES / name)
            out = tmp_path / name
            E.write_grid(g, out)
            assert out.read_bytes() == (FILES / name).read_bytes()
            assert g.values.dtype == np.float64

    def test_coefficient_file_matches_oracle(self, tmp_path):
        g = E.read_grid(FILES / "g3d.eccg")
        cg = E.read_coefficients(FILES / "c3d.eccg")
        assert cg.coeffs.dtype == np.int8
        assert np.array_equal(cg.coeffs, oracle.coefficients(g.values))
        E.write_coefficients(cg, tmp_path / "c.eccg")
        assert (tmp_path / "c.eccg").read_bytes() == (FILES / "c3d.eccg").read_bytes()

    def test_curve_files(self, tmp_path):
        g = E.read_grid(FILES / "g3d.eccg")
        c = E.read_curve(FILES / "curve_g3d_32.csv")
        assert c.is_integral
        ts = E.thresholds_from_range(float(g.values.min()), float(g.values.max()), 32)   # grid.py:192-196
        assert np.array_equal(c.taus, ts.taus)
        assert np.array_equal(c.values, oracle.curve(g.values, ts.taus))
        for name in ("curve_g3d_32.csv", "soft_g2d_16.csv"):
            back = E.read_curve(FILES / name)
            E.write_curve(back, tmp_path / name)
            assert (tmp_path / name).read_bytes() == (FILES / name).read_bytes()
        assert not E.read_curve(FILES / "soft_g2d_16.csv").is_integral


class TestFormatErrors:
    """grid.py:235-278 semantics, mirroring the reference's test_grid.py cases."""

    def _file(self, tmp_path, arr=None):
        path = tmp_path / "g.eccg"
        E.write_grid(E.ScalarGrid(np.zeros((2, 2)) if arr is None else arr), path)
        return path

    def test_header_layout(self, tmp_path):
        path = tmp_path / "g.eccg"
        E.write_grid(E.ScalarGrid([[5.0]]), path)
        blob = path.read_bytes()
        assert blob[:4] == E.MAGIC and blob[4] == 1 and blob[5] == 2 and blob[6:8] == b"\x00\x00"
        assert len(blob) == 8 + 16 + 4

    @pytest.mark.parametrize("pos,val", [(0, 0x00), (4, 9), (5, 4), (6, 1)])
    def test_header_corruptions_are_format_errors(self, tmp_path, pos, val):
        path = self._file(tmp_path)
        blob = _blob(path)
        blob[pos] = val if pos else blob[0] ^ 0xFF
        path.write_bytes(bytes(blob))
        with pytest.raises(E.FormatError):
            E.read_grid(path)
        with pytest.raises(E.FormatError):
            E.load_grid_device(path, "cpu")

    def test_short_and_truncated(self, tmp_path):
        path = self._file(tmp_path)
        path.write_bytes(path.read_bytes()[:5])
        with pytest.raises(E.FormatError):
            E.read_grid(path)
        path = self._file(tmp_path)
        path.write_bytes(path.read_bytes()[:12])
        with pytest.raises(E.FormatError):
            E.read_grid(path)

    def test_payload_mismatch_is_corruption(self, tmp_path):
        path = self._file(tmp_path, np.zeros((4, 4)))
        path.write_bytes(path.read_bytes()[:-4])
        with pytest.raises(E.CorruptionError):
            E.read_grid(path)
        with pytest.raises(E.CorruptionError):
            E.load_grid_device(path, "cpu")
        path = self._file(tmp_path)
        blob = _blob(path)
        blob[8] = 3
        path.write_bytes(bytes(blob))
        with pytest.raises(E.CorruptionError):
            E.read_grid(path)

    def test_zero_extent(self, tmp_path):
        path = self._file(tmp_path)
        blob = _blob(path)
        blob[8] = 0
        path.write_bytes(bytes(blob))
        with pytest.raises(E.FormatError):
            E.read_grid(path)

    def test_non_finite_payload(self, tmp_path):
        path = self._file(tmp_path)
        blob = _blob(path)
        blob[-4:] = np.array([np.nan], dtype="<f4").tobytes()
        path.write_bytes(bytes(blob))
        with pytest.raises(ValueError):
            E.read_grid(path)
        with pytest.raises(ValueError):
            E.load_grid_device(path, "cpu")

    def test_missing_file(self, tmp_path):
        with pytest.raises(OSError):
            E.read_grid(tmp_path / "nope.eccg")

    def test_coefficient_files(self, tmp_path, rng):
        path = tmp_path / "c.eccg"
        E.write_coefficients(E.CoefficientGrid(oracle.coefficients(np.zeros((2, 2)))), path)
        assert path.read_bytes()[4] == 2
        with pytest.raises(E.FormatError):
            E.read_grid(path)
        blob = _blob(path)
        blob[-4:] = np.array([99], dtype="<i4").tobytes()
        path.write_bytes(bytes(blob))
        with pytest.raises(E.CorruptionError):
            E.read_coefficients(path)

    def test_curve_header_required(self, tmp_path):
        path = tmp_path / "c.csv"
        path.write_text("tau,chi\n0.5,1\n")
        with pytest.raises(E.FormatError):
            E.read_curve(path)


class TestLoader:
    def test_cpu_planes_and_chunks(self, tmp_path, rng):
        x = rng.random((7, 5, 6)).astype(np.float32)
        path = tmp_path / "g.eccg"
        E.write_grid(x, path)
        assert np.array_equal(E.load_grid_device(path, "cpu").numpy(), x)
        assert np.array_equal(E.load_grid_device(path, "cpu", planes=(2, 5)).numpy(), x[2:5])
        assert E.load_grid_device(path, "cpu", planes=(3, 3)).shape == (0, 5, 6)
        with pytest.raises(ValueError):
            E.load_grid_device(path, "cpu", planes=(4, 9))

    def test_slabs_carry_neighbour_planes(self, tmp_path, rng):
        x = rng.random((10, 4, 8)).astype(np.float32)
        path = tmp_path / "g.eccg"
        E.write_grid(x, path)
        world = 3
        for rank in range(world):
            padded, (z0, z1) = E.load_slab_device(path, rank, world, "cpu")
            assert padded.shape == (z1 - z0 + 2, 4, 8)
            assert np.array_equal(padded[1:-1].numpy(), x[z0:z1])
            if z0 > 0:
                assert np.array_equal(padded[0].numpy(), x[z0 - 1])
            if z1 < 10:
                assert np.array_equal(padded[-1].numpy(), x[z1])


@pytest.mark.gpu
class TestLoaderGPU:
    def test_streamed_load_matches_file(self, tmp_path, rng):
        x = rng.random((33, 40, 44)).astype(np.float32)
        path = tmp_path / "g.eccg"
        E.write_grid(x, path)
        for chunk in (4096, 40 * 44 * 4 * 3 + 12, 64 << 20):
            t = E.load_grid_device(path, chunk_bytes=chunk)
            assert t.is_cuda and np.array_equal(t.cpu().numpy(), x)
        t = E.load_grid_device(path, planes=(5, 29), chunk_bytes=5000)
        assert np.array_equal(t.cpu().numpy(), x[5:29])

    def test_file_backed_slabs_histogram(self, tmp_path, rng):
        """Slabs loaded from a file (own planes + neighbour planes, no halo
        exchange) sum to the whole volume's histogram, bit-exact."""
        from paper_2510_20271_b200 import _lib

        x = rng.random((23, 35, 72)).astype(np.float32)
        path = tmp_path / "g.eccg"
        E.write_grid(x, path)
        ts = E.ThresholdSet(np.linspace(0.0, 1.0, 129)[1:])
        total = np.zeros(129, np.int64)
        world = 4
        for rank in range(world):
            padded, (z0, z1) = E.load_slab_device(path, rank, world)
            lo = 1 if rank == 0 else 0
            hi = padded.shape[0] - (1 if rank == world - 1 else 0)
            view = padded[lo:hi]
            table, binning = ts.device_table(_lib.DTYPE_F32, view.device)
            hist = torch.empty(129, dtype=torch.int64, device="cuda")
            d = _lib.dims_arg(view.shape)
            _lib.check(_lib.lib().ecc_histogram_range(_lib.ptr(view), _lib.DTYPE_F32, 3, _lib.ptr(d), 1, 1 - lo,
                                                      1 - lo + z1 - z0, _lib.ptr(table),
                                                      _lib.ctypes.byref(binning), _lib.ptr(hist),
                                                      _lib.stream_ptr(view)))
            total += hist.cpu().numpy()
        assert np.array_equal(total, np.append(*oracle.histogram(x, ts.taus)))

"""The ``ecc`` command line (ecckit cli.py), mirroring the reference's
test_cli.py: CPU tests for generation, argument handling and error paths;
GPU tests for the compute / soft / gradcheck / coeffs / bench commands."""

from __future__ import annotations

import json

import numpy as np
import pytest

import paper_2510_20271_b200 as E
from paper_2510_20271_b200 import cli
from oracle import oracle


@pytest.fixture
def grid_file(tmp_path):
    path = tmp_path / "g.eccg"
    assert cli.main(["generate", "--dims", "24x20", "--seed", "3", "--output", str(path)]) == 0
    return path


class TestGenerate:
    def test_uniform_random_is_pcg64_float32(self, grid_file):
        g = E.read_grid(grid_file)
        want = np.random.default_rng(3).random((24, 20)).astype(np.float32)
        assert np.array_equal(g.values, want.astype(np.float64))

    def test_kinds_and_3d(self, tmp_path):
        for kind in ("gaussian-blobs", "radial-gradient"):
            path = tmp_path / f"{kind}.eccg"
            assert cli.main(["generate", "--kind", kind, "--dims", "6x7x8", "--output", str(path)]) == 0
            g = E.read_grid(path)
            assert g.dims == (6, 7, 8) and 0.0 <= g.values.min() and g.values.max() <= 1.0

    def test_seed_reproducible(self, tmp_path):
        a, b = tmp_path / "a.eccg", tmp_path / "b.eccg"
        for p in (a, b):
            cli.main(["generate", "--dims", "9x9", "--seed", "11", "--output", str(p)])
        assert a.read_bytes() == b.read_bytes()

    def test_bad_dims_rejected(self, tmp_path):
        with pytest.raises(SystemExit):
            cli.main(["generate", "--dims", "9", "--output", str(tmp_path / "x.eccg")])

    def test_malformed_input_fails_cleanly(self, tmp_path, capsys):
        bad = tmp_path / "bad.eccg"
        bad.write_bytes(b"nope")
        rc = cli.main(["coeffs", "--input", str(bad), "--output", str(tmp_path / "c.eccg")])
        assert rc == 2 and "error:" in capsys.readouterr().err

    def test_checksum_is_order_sensitive(self):
        c1 = E.EulerCurve([0.1, 0.2], np.array([1, 2], np.int64))
        c2 = E.EulerCurve([0.1, 0.2], np.array([2, 1], np.int64))
        assert cli.curve_checksum(c1) != cli.curve_checksum(c2)
        assert cli.curve_checksum(c1) == cli.curve_checksum(E.EulerCurve([0.1, 0.2], np.array([1, 2], np.int64)))


@pytest.mark.gpu
class TestCommandsGPU:
    def test_compute_and_timing(self, grid_file, tmp_path):
        out, timing = tmp_path / "c.csv", tmp_path / "t.json"
        assert cli.main(["compute", "--input", str(grid_file), "--bins", "32", "--output", str(out),
                         "--emit-timing", str(timing)]) == 0
        curve = E.read_curve(out)
        x = E.read_grid(grid_file).values
        assert np.array_equal(curve.values, oracle.curve(x, curve.taus))
        t = json.loads(timing.read_text())
        assert t["bins"] == 32 and t["dims"] == [24, 20] and t["wall_ms"] > 0

    def test_taus_file_and_strategy(self, grid_file, tmp_path):
        taus = tmp_path / "taus.csv"
        taus.write_text("threshold\n0.25\n0.5\n0.75\n")
        out = tmp_path / "c.csv"
        assert cli.main(["compute", "--input", str(grid_file), "--taus", str(taus), "--strategy", "chunked:7",
                         "--workers", "4", "--output", str(out)]) == 0
        assert np.array_equal(E.read_curve(out).taus, [0.25, 0.5, 0.75])

    def test_soft_and_coeffs(self, grid_file, tmp_path):
        out = tmp_path / "s.csv"
        assert cli.main(["soft", "--input", str(grid_file), "--bins", "16", "--lambda", "20", "--alpha", "0.3",
                         "--direction", "1,2", "--output", str(out)]) == 0
        assert not E.read_curve(out).is_integral
        cfile = tmp_path / "c.eccg"
        assert cli.main(["coeffs", "--input", str(grid_file), "--output", str(cfile)]) == 0
        x = E.read_grid(grid_file).values
        assert np.array_equal(E.read_coefficients(cfile).coeffs, oracle.coefficients(x))

    def test_gradcheck_report(self, grid_file, tmp_path):
        rep = tmp_path / "r.json"
        rc = cli.main(["gradcheck", "--input", str(grid_file), "--lambda", "8", "--alpha", "0.2", "--bins", "8",
                       "--report", str(rep)])
        r = json.loads(rep.read_text())
        assert {"d_values", "d_tau", "d_u", "tangency", "pass"} <= set(r)
        assert rc == (0 if r["pass"] else 1)
        assert max(r["normwise"].values()) <= 1e-4

    def test_bench_gate(self, tmp_path, capsys):
        rep = tmp_path / "b.json"
        assert cli.main(["bench", "--sizes", "40x36,20x24x28", "--bins", "64", "--repeats", "2",
                         "--report", str(rep), "--csv", str(tmp_path / "b.csv")]) == 0
        rows = json.loads(rep.read_text())["rows"]
        assert len(rows) == 2 * len(cli.VARIANTS) and len({r["checksum"] for r in rows if r["dims"] == [40, 36]}) == 1


def test_generators_match_reference_files(tmp_path):
    """generate writes the same bytes as the reference's generator (golden files)."""
    from pathlib import Path

    files = Path(__file__).resolve().parent / "golden" / "files"
    for name, argv in (("blobs_12x10_s4_b3.eccg", ["--kind", "gaussian-blobs", "--dims", "12x10", "--seed", "4",
                                                   "--blobs", "3"]),
                       ("radial_5x6x7.eccg", ["--kind", "radial-gradient", "--dims", "5x6x7"]),
                       ("uniform_4x5x6_s9.eccg", ["--dims", "4x5x6", "--seed", "9"])):
        out = tmp_path / name
        assert cli.main(["generate", *argv, "--output", str(out)]) == 0
        assert out.read_bytes() == (files / name).read_bytes(), name

"""Host-side mirror of the reference API: validation and pure-host helpers
behave like ecckit (test_grid.py, test_hard.py:53-123, test_soft.py:114-293)
without touching the GPU."""

import numpy as np
import pytest

import paper_2510_20271_b200 as E


class TestTypes:
    def test_scalar_grid_validation(self):
        g = E.ScalarGrid([[0.0, 1.0], [2.0, 3.0]])
        assert g.dims == (2, 2) and g.ndim == 2 and g.size == 4
        with pytest.raises(ValueError):
            g.values[0, 0] = 1.0
        for bad in (np.zeros(5), np.zeros((2, 2, 2, 2)), [[np.nan, 0.0]], [[np.inf, 0.0]]):
            with pytest.raises(ValueError):
                E.ScalarGrid(bad)

    def test_threshold_set_validation(self):
        for bad in ([], [1.0, 1.0], [2.0, 1.0], [0.0, np.inf]):
            with pytest.raises(ValueError):
                E.ThresholdSet(bad)

    def test_bin_index(self):
        ts = E.ThresholdSet([1.0, 2.0, 3.0])
        assert E.bin_index(1.0, ts) == 0
        assert E.bin_index(3.0 + 1e-12, ts) is None
        assert E.bin_index(1.5, ts) == 1 and E.bin_index(0.0, ts) == 0

    def test_merge_histograms(self):
        t = np.array([0.0, 1.0])
        a = E.HistogramBins(t, np.array([1, 2]), 3)
        b = E.HistogramBins(t, np.array([-1, 5]), -2)
        m = E.merge_histograms([a, b])
        assert np.array_equal(m.bins, [0, 7]) and m.overflow == 1
        with pytest.raises(ValueError):
            E.merge_histograms([])
        with pytest.raises(ValueError):
            E.merge_histograms([a, E.HistogramBins(np.array([0.0]), np.array([1]), 0)])
        with pytest.raises(ValueError):
            E.merge_histograms([a, E.HistogramBins(np.array([0.0, 2.0]), np.array([1, 2]), 0)])

    def test_parse_strategy(self):
        assert E.parse_strategy("fullsweep") == E.FullSweep()
        assert E.parse_strategy("chunked:64") == E.Chunked(64)
        for bad in ("sideways", "chunked:0"):
            with pytest.raises(ValueError):
                E.parse_strategy(bad)

    def test_thresholds_from_range(self):
        assert np.array_equal(E.thresholds_from_range(0.0, 10.0, 2).taus, [5.0, 10.0])
        assert np.array_equal(E.thresholds_from_range(4.25, 4.25, 8).taus, [4.25])
        with pytest.raises(ValueError):
            E.uniform_thresholds(E.ScalarGrid([[1.0]]), 0)

    def test_curve_type(self):
        c = E.EulerCurve([0.0, 1.0], np.array([0, 1], dtype=np.int64))
        assert c.is_integral and len(c) == 2
        with pytest.raises(ValueError):
            E.EulerCurve([0.0], np.array([0, 1]))


class TestSoftHost:
    def test_params_validation(self):
        t = E.ThresholdSet([0.0])
        with pytest.raises(ValueError):
            E.SoftEccParams(lam=0.0, alpha=0.0, u=np.array([1.0, 0.0]), taus=t)
        with pytest.raises(ValueError):
            E.SoftEccParams(lam=1.0, alpha=0.0, u=np.array([1.0, 1.0]), taus=t)

    def test_pixel_coordinates(self):
        c = E.pixel_coordinates((3, 5))
        assert c.shape == (15, 2) and c.min() == -1.0 and c.max() == 1.0
        assert (E.pixel_coordinates((1, 4))[:, 0] == 0.0).all()
        assert np.array_equal(E.pixel_coordinates((4, 3, 2), 5, 17), E.pixel_coordinates((4, 3, 2))[5:17])

    def test_reparametrization(self, rng):
        assert np.allclose(E.reparametrize_direction([3.0, 4.0]), [0.6, 0.8], rtol=0, atol=1e-15)
        with pytest.raises(ValueError):
            E.reparametrize_direction([1e-13, 0.0])
        for _ in range(10):
            v = rng.normal(size=3) * rng.uniform(0.5, 3)
            dv = rng.normal(size=3)
            step = 1e-6
            fd = (E.reparametrize_direction(v + step * dv) - E.reparametrize_direction(v - step * dv)) / (2 * step)
            assert np.abs(E.reparametrize_direction_jvp(v, dv) - fd).max() / max(np.abs(fd).max(), 1e-9) <= 1e-6

    def test_module_construction(self):
        m = E.SoftECC(np.linspace(0, 1, 8), [1.0, 2.0], alpha=0.3, lam=50.0)
        assert m.taus.shape == (8,) and m.v.shape == (2,) and float(m.lam) == 50.0
        u = m.direction().detach().numpy()
        assert abs(np.linalg.norm(u) - 1) < 1e-12
        with pytest.raises(ValueError):
            E.SoftECC([0.0], [0.0, 0.0])
        with pytest.raises(ValueError):
            E.SoftECC([0.0], [1.0, 0.0], lam=-1.0)


def test_engine_fails_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError):
        E.compute_ecc(E.ScalarGrid([[1.0, 2.0]]), E.ThresholdSet([1.0, 2.0]))


def test_band_window_condition():
    """The windowed soft kernels' condition (soft.band_window mirrors
    ecc_soft.cu band_ok): C3's / C4's thresholds get a 128-threshold window;
    unsorted, too dense for the window, too few or too many thresholds, or
    a soft sigmoid (small lambda) fall back to all thresholds."""
    from paper_2510_20271_b200.soft import band_window

    span = 0.3 * (3.0 / np.sqrt(5.0))
    taus = np.linspace(-span, 1.0 + span, 257)[1:]
    assert band_window(taus, 50.0) == 128
    assert band_window(taus[::-1], 50.0) == 256               # unsorted
    assert band_window(taus, 5.0) == 256                      # W = 24 ln2 / lam wider than 7 blocks
    assert band_window(np.linspace(0, 1, 64), 50.0) == 64     # fewer than NWB + 2 blocks
    assert band_window(np.linspace(0, 1, 1024), 500.0) == 1024   # more than 16 bands
    assert band_window(np.linspace(0, 1, 368), 500.0) == 128


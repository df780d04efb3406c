"""Discrete ECC on the GPU: bit-exact parity with the reference (golden vectors)
and with the CPU oracle, through the reference-shaped API and the C ABI.

Mirrors the reference's tests/test_hard.py, test_coefficients.py and
acceptance criteria 1/3/6 (test_acceptance.py:51-209) with the CUDA engine
in place of ecckit's numpy kernels.
"""

import numpy as np
import pytest
import torch
from hypothesis import given, settings
from hypothesis import strategies as st

from conftest import golden_cases, random_f32_grid, random_int_grid
from oracle import oracle

pytestmark = pytest.mark.gpu

E = pytest.importorskip("paper_2510_20271_b200")


def _grid(vals):
    return E.ScalarGrid(vals)


class TestGoldenParity:
    def test_coefficients(self, golden):
        for k in golden_cases(golden, "coeff"):
            x = golden[f"coeff{k}_x"]
            got = E.compute_coefficients(_grid(x)).coeffs
            assert np.array_equal(got, golden[f"coeff{k}_c"]), f"case {k} dims {x.shape}"

    def test_coefficients_all_dtypes(self, golden):
        dev = torch.device("cuda")
        for k in golden_cases(golden, "coeff"):
            x = golden[f"coeff{k}_x"]
            want = golden[f"coeff{k}_c"]
            for dt in (torch.float64, torch.float32):
                t = torch.from_numpy(x).to(dev, dt)
                if dt == torch.float32 and not np.array_equal(t.double().cpu().numpy(), x):
                    continue
                assert np.array_equal(E.coefficients_device(t).cpu().numpy(), want), (k, dt)

    def test_histograms_and_curves(self, golden):
        for k in golden_cases(golden, "hist"):
            x = golden[f"hist{k}_x"]
            ts = E.ThresholdSet(golden[f"hist{k}_taus"])
            g = _grid(x)
            h = E.accumulate_histogram(g, ts)
            assert np.array_equal(h.bins, golden[f"hist{k}_bins"]), f"case {k} {x.shape}"
            assert h.overflow == int(golden[f"hist{k}_overflow"][0]), f"case {k}"
            curve = E.compute_ecc(g, ts)
            assert curve.values.dtype == np.int64
            assert np.array_equal(curve.values, golden[f"hist{k}_curve"]), f"case {k}"

    def test_histograms_every_dtype(self, golden):
        """float64 and float32 device tensors (and uint8 when exact) agree."""
        dev = torch.device("cuda")
        for k in golden_cases(golden, "hist"):
            x = golden[f"hist{k}_x"]
            ts = E.ThresholdSet(golden[f"hist{k}_taus"])
            want = np.concatenate([golden[f"hist{k}_bins"], golden[f"hist{k}_overflow"]])
            variants = [torch.from_numpy(x).to(dev)]
            if np.array_equal(x.astype(np.float32).astype(np.float64), x):
                variants.append(torch.from_numpy(x.astype(np.float32)).to(dev))
            if x.min() >= 0 and x.max() <= 255 and np.array_equal(np.floor(x), x):
                variants.append(torch.from_numpy(x.astype(np.uint8)).to(dev))
            for t in variants:
                got = E.histogram_device(t, ts)[0].cpu().numpy()
                assert np.array_equal(got, want), (k, t.dtype)

    def test_uniform_thresholds(self, golden):
        for k in golden_cases(golden, "uthr"):
            x = golden[f"uthr{k}_x"]
            bins = int(golden[f"uthr{k}_bins"][0])
            got = E.uniform_thresholds(_grid(x), bins).taus
            assert np.array_equal(got, golden[f"uthr{k}_taus"]), k


class TestFixtures:
    """test_hard.py:27-50, test_coefficients.py:29-69."""

    def test_center_peak_2d(self):
        vals = np.zeros((3, 3))
        vals[1, 1] = 1.0
        assert np.array_equal(E.compute_ecc(_grid(vals), E.ThresholdSet([0.0, 1.0])).values, [0, 1])

    def test_center_peak_3d_shell(self):
        vals = np.zeros((3, 3, 3))
        vals[1, 1, 1] = 1.0
        assert np.array_equal(E.compute_ecc(_grid(vals), E.ThresholdSet([0.0, 1.0])).values, [2, 1])

    def test_threshold_below_min_gives_zero(self, rng):
        x = random_f32_grid(rng, 2, 8)
        curve = E.compute_ecc(_grid(x), E.ThresholdSet([x.min() - 1.0, x.max()]))
        assert curve.values[0] == 0 and curve.values[-1] == 1

    def test_tail_is_one_at_max(self, rng):
        for _ in range(10):
            x = random_int_grid(rng, 2, 10)
            g = _grid(x)
            assert E.compute_ecc(g, E.uniform_thresholds(g, 7)).values[-1] == 1

    def test_single_pixel_and_2x2(self):
        assert np.array_equal(E.compute_coefficients(_grid([[5.0]])).coeffs, [[1]])
        assert np.array_equal(E.compute_coefficients(_grid(np.zeros((2, 2)))).coeffs.ravel(), [1, 0, 0, 0])


class TestOracleEquivalence:
    def test_random_int_grids(self, rng):
        """acceptance criterion 1 (test_acceptance.py:51-68): 200 grids, every distinct value."""
        for ndim, max_extent in ((2, 32), (3, 8)):
            for _ in range(100):
                x = random_int_grid(rng, ndim, max_extent)
                taus = np.unique(x)
                got = E.compute_ecc(_grid(x), E.ThresholdSet(taus)).values
                assert np.array_equal(got, oracle.curve(x, taus)), x.shape

    def test_float_plateaus(self, rng):
        vals = rng.random((9, 9)).astype(np.float32).astype(np.float64)
        vals[vals < 0.4] = 0.25
        taus = np.unique(vals)
        assert np.array_equal(E.compute_ecc(_grid(vals), E.ThresholdSet(taus)).values, oracle.curve(vals, taus))

    @given(st.lists(st.integers(1, 4), min_size=2, max_size=3), st.data())
    @settings(max_examples=200, deadline=None)
    def test_arbitrary_float32_property(self, dims, data):
        """test_hard.py:169-188: arbitrary float32 values incl. +-0 and subnormals."""
        n = int(np.prod(dims))
        values = data.draw(st.lists(st.floats(allow_nan=False, allow_infinity=False, width=32),
                                     min_size=n, max_size=n))
        x = np.array(values, dtype=np.float64).reshape(dims)
        taus = np.unique(x)
        got = E.compute_ecc(_grid(x), E.ThresholdSet(taus)).values
        assert np.array_equal(got, oracle.curve(x, taus))

    def test_odd_shapes_and_sizes(self, rng):
        """Tile edges: extents around multiples of the 32x16 tile and z-chunks."""
        for dims in [(37, 23), (9, 8, 7), (1, 1), (1, 200), (200, 1), (33, 17), (31, 65), (3, 1, 1), (1, 1, 50),
                     (70, 33, 17), (130, 5, 40), (2, 300, 3)]:
            x = rng.random(dims).astype(np.float32).astype(np.float64)
            g = _grid(x)
            ts = E.uniform_thresholds(g, 97)
            assert np.array_equal(E.compute_ecc(g, ts).values, oracle.curve(x, ts.taus)), dims
            assert np.array_equal(E.compute_coefficients(g).coeffs, oracle.coefficients(x)), dims

    def test_mass_is_one_with_overflow(self, rng):
        for trial in range(20):
            x = random_int_grid(rng, 2 if trial % 2 else 3, 10 if trial % 2 else 5)
            hi = float(x.max())
            ts = E.ThresholdSet([hi / 3, hi / 2]) if hi > 0 else E.ThresholdSet([0.0])
            h = E.accumulate_histogram(_grid(x), ts)
            assert int(h.bins.sum()) + h.overflow == 1

    def test_medium_volume_vs_oracle(self):
        """uniform-random 3D with 1024 bins, several z-chunks and tiles."""
        x = oracle.counter_grid(7, (96, 80, 72)).reshape(96, 80, 72)
        t = torch.from_numpy(x).cuda()
        lo, hi, bad = E.device_minmax(t)
        assert bad == 0 and lo == float(x.min()) and hi == float(x.max())
        ts = E.thresholds_from_range(lo, hi, 1024)
        curve, hist = E.ecc_discrete(t, ts, return_hist=True)
        bins, ovf = oracle.histogram(x, ts.taus)
        assert np.array_equal(hist.cpu().numpy(), np.append(bins, ovf))
        assert np.array_equal(curve.cpu().numpy(), np.cumsum(bins))


class TestBatchedAndValidation:
    def test_batched_matches_individual(self, rng):
        xs = rng.random((5, 19, 23, 11)).astype(np.float32)
        ts = E.ThresholdSet(np.linspace(0.05, 0.95, 33))
        curves = E.ecc_discrete(torch.from_numpy(xs).cuda(), ts, ndim=3).cpu().numpy()
        for i in range(5):
            assert np.array_equal(curves[i], oracle.curve(xs[i], ts.taus))
        xs2 = rng.integers(0, 256, (4, 40, 50)).astype(np.uint8)
        taus2 = np.arange(0.0, 256.0, 3.0)
        curves2 = E.ecc_discrete(torch.from_numpy(xs2).cuda(), E.ThresholdSet(taus2), ndim=2).cpu().numpy()
        for i in range(4):
            assert np.array_equal(curves2[i], oracle.curve(xs2[i].astype(np.float64), taus2))

    def test_bad_workers_and_strategy(self, rng):
        g = _grid(random_int_grid(rng, 2, 4))
        with pytest.raises(ValueError):
            E.compute_ecc(g, E.uniform_thresholds(g, 2), E.FullSweep(), 0)
        with pytest.raises(TypeError):
            E.compute_ecc(g, E.uniform_thresholds(g, 2), "sideways")

    def test_strategies_and_workers_identical(self, rng):
        x = random_int_grid(rng, 3, 6)
        g = _grid(x)
        ts = E.uniform_thresholds(g, 9)
        ref = E.compute_ecc(g, ts).values
        for strategy in (E.FullSweep(), E.Chunked(1), E.Chunked(7)):
            for workers in (1, 2, 8):
                assert E.compute_ecc(g, ts, strategy, workers).values.tobytes() == ref.tobytes()

    def test_nonfinite_device_grid_rejected(self):
        t = torch.zeros((4, 4), device="cuda")
        t[1, 2] = float("nan")
        with pytest.raises(ValueError):
            E.ScalarGrid(t)

    def test_c1_uint8(self):
        """BASELINE configs[0]: 256x256 uint8, 256 thresholds, bit-exact."""
        x = np.random.default_rng(1).integers(0, 256, (256, 256), np.uint8)
        t = torch.from_numpy(x).cuda()
        lo, hi, _ = E.device_minmax(t)
        ts = E.thresholds_from_range(lo, hi, 256)
        got = E.ecc_discrete(t, ts).cpu().numpy()
        assert np.array_equal(got, oracle.curve(x.astype(np.float64), ts.taus))


class TestFastPath:
    """The bit-sliced TMA kernels (float32, W % 4 == 0) against the oracle and
    against the generic sweep, on shapes that hit every tile/segment edge.

    The default kernel works on the bin image (per-voxel coefficients in the
    order (bin, index), a different but equally valid total order), so its
    per-bin sums, not its coefficients, are what must match the reference."""

    SHAPES = [(1, 4, 4), (3, 5, 8), (7, 31, 32), (9, 30, 36), (5, 61, 100), (33, 33, 128), (2, 64, 132),
              (17, 90, 260), (64, 31, 4), (1, 1, 64), (40, 1, 40), (65, 47, 68)]

    KERNELS = {"bin": {}, "value": {"f3": "value"}, "branch": {"f3": "branch"}, "cta": {"f3": "cta"},
               "rank2": {"f3": "rank2"}, "no2d": {"f3": "no2d"}, "dyn4": {"zunit": 4}, "dyn7": {"zunit": 7},
               "edge1": {"f3": "edge1"}, "dummy": {"f3": "dummy"}, "static": {"f3": "static"},
               "generic": {"generic": 1}}

    @classmethod
    def _all(cls, t, ts, **kw):
        """Histogram through each kernel: the rank4 TMA kernel (default when
        the thresholds have an edge table), its variants, the value-order TMA
        kernel and the generic sweep."""
        from paper_2510_20271_b200 import _lib

        out = {}
        for name, var in cls.KERNELS.items():
            with _lib.variant(**var):
                out[name] = E.histogram_device(t, ts, **kw).cpu().numpy()
        return out

    @classmethod
    def _both(cls, t, ts, **kw):
        out = cls._all(t, ts, **kw)
        for name in ("value", "branch", "cta", "rank2", "no2d", "dyn4", "dyn7", "edge1", "dummy", "static"):
            assert np.array_equal(out[name], out["bin"]), name
        return out["bin"], out["generic"]

    def test_random_volumes(self, rng):
        for dims in self.SHAPES:
            x = rng.random(dims).astype(np.float32)
            t = torch.from_numpy(x).cuda()
            for nb in (1, 7, 256, 1024):
                lo, hi = float(x.min()), float(x.max())
                ts = E.thresholds_from_range(lo, hi, nb)
                fast, gen = self._both(t, ts)
                want = np.append(*oracle.histogram(x, ts.taus))
                assert np.array_equal(fast[0], want), (dims, nb)
                assert np.array_equal(gen[0], want), (dims, nb)

    def test_ties_signed_zeros_subnormals(self, rng):
        specials = np.array([0.0, -0.0, 1e-45, -1e-45, 1.17549435e-38, -1.4e-45, 3.4e38, -3.4e38, 1.0, -1.0, 0.5],
                            dtype=np.float32)
        for dims in [(6, 9, 12), (11, 40, 36), (4, 33, 64)]:
            for pool in (specials, np.array([0.0, 1.0, 2.0], np.float32)):
                x = rng.choice(pool, size=dims).astype(np.float32)
                t = torch.from_numpy(x).cuda()
                taus = np.unique(x.astype(np.float64))
                ts = E.ThresholdSet(taus)
                fast, _ = self._both(t, ts)
                want = np.append(*oracle.histogram(x, taus))
                assert np.array_equal(fast[0], want), dims
                c = np.cumsum(want[:-1])
                assert c[-1] == 1

    def test_hostile_thresholds_binary_search_path(self, rng):
        x = (rng.normal(0, 3, (9, 20, 24))).astype(np.float32)
        t = torch.from_numpy(x).cuda()
        for taus in (np.unique(rng.normal(0, 2, 300)), np.array([-1e300, 0.0, 1e300]),
                     np.array([-1.0, -1e-45, 0.0, 1e-45, 0.5])):
            ts = E.ThresholdSet(taus)
            fast, gen = self._both(t, ts)
            want = np.append(*oracle.histogram(x, taus))
            assert np.array_equal(fast[0], want) and np.array_equal(gen[0], want)

    def test_batched(self, rng):
        from paper_2510_20271_b200 import _lib

        xs = rng.random((3, 10, 37, 44)).astype(np.float32)
        ts = E.ThresholdSet(np.linspace(0.01, 0.99, 129))
        for zunit in (0, 3):   # static partition, dynamic work queue (units span items)
            with _lib.variant(zunit=zunit):
                h = E.histogram_device(torch.from_numpy(xs).cuda(), ts, ndim=3).cpu().numpy()
            for i in range(3):
                assert np.array_equal(h[i], np.append(*oracle.histogram(xs[i], ts.taus))), (zunit, i)

    def test_plane_range_slabs(self, rng):
        """ecc_histogram_range: slabs with halos sum to the whole volume (C5 path)."""
        from paper_2510_20271_b200 import _lib

        D, H, W = 23, 35, 72
        x = rng.random((D, H, W)).astype(np.float32)
        ts = E.ThresholdSet(np.linspace(0.0, 1.0, 65)[1:])
        t = torch.from_numpy(x).cuda()
        table, binning = ts.device_table(_lib.DTYPE_F32, t.device)
        want = np.append(*oracle.histogram(x, ts.taus))
        for zunit in (0, 2, 3):   # static partition and the dynamic work queue
            with _lib.variant(zunit=zunit):
                total = np.zeros(65, np.int64)
                for z0, z1 in [(0, 7), (7, 8), (8, 16), (16, 23)]:
                    lo, hi = max(0, z0 - 1), min(D, z1 + 1)
                    view = t[lo:hi]
                    hist = torch.empty(65, dtype=torch.int64, device="cuda")
                    d = _lib.dims_arg(view.shape)
                    _lib.check(_lib.lib().ecc_histogram_range(_lib.ptr(view), _lib.DTYPE_F32, 3, _lib.ptr(d), 1,
                                                              z0 - lo, z1 - lo, _lib.ptr(table),
                                                              _lib.ctypes.byref(binning), _lib.ptr(hist),
                                                              _lib.stream_ptr(view)))
                    total += hist.cpu().numpy()
            assert np.array_equal(total, want), zunit

    def test_large_volume_invariants(self):
        """256^3 counter grid: bit-exact vs oracle, sum c = 1, tail = 1."""
        dims = (256, 256, 256)
        from paper_2510_20271_b200 import _lib

        t = torch.empty(dims, dtype=torch.float32, device="cuda")
        _lib.check(_lib.lib().ecc_counter_grid(9, 0, t.numel(), _lib.ptr(t), _lib.stream_ptr(t)))
        x = t.cpu().numpy()
        assert np.array_equal(x.ravel(), oracle.counter_grid(9, dims))
        lo, hi, _ = E.device_minmax(t)
        ts = E.thresholds_from_range(lo, hi, 1024)
        curve, hist = E.ecc_discrete(t, ts, return_hist=True)
        h = hist.cpu().numpy()
        assert int(h.sum()) == 1 and int(curve[-1]) == 1
        assert np.array_equal(h, np.append(*oracle.histogram(x, ts.taus)))


class TestFastPath2D:
    def test_2d_images_fast_path(self, rng):
        """2D float32 images take the TMA kernel with D = 1 (W % 4 == 0)."""
        xs = rng.random((3, 70, 132)).astype(np.float32)
        ts = E.ThresholdSet(np.linspace(0.0, 1.0, 257)[1:])
        curves = E.ecc_discrete(torch.from_numpy(xs).cuda(), ts, ndim=2).cpu().numpy()
        for i in range(3):
            assert np.array_equal(curves[i], oracle.curve(xs[i], ts.taus))

    def test_large_uint8_volume_generic_path(self, rng):
        x = rng.integers(0, 256, (40, 64, 61), dtype=np.uint8)
        ts = E.ThresholdSet(np.arange(0.0, 256.0, 5.0))
        got = E.ecc_discrete(torch.from_numpy(x).cuda(), ts).cpu().numpy()
        assert np.array_equal(got, oracle.curve(x.astype(np.float64), ts.taus))


class TestBinKernelLimits:
    """The bin-image kernel takes nb <= 8190 (16-bit lanes hold 4 * bin); larger
    threshold sets fall back to the value-order kernel.  Both sides of the
    limit, and non-power-of-two cell tables, stay bit-exact."""

    @pytest.mark.parametrize("nb", [1000, 4097, 8190, 8191, 12000])
    def test_many_bins(self, rng, nb):
        x = rng.random((20, 45, 132)).astype(np.float32)
        t = torch.from_numpy(x).cuda()
        ts = E.thresholds_from_range(float(x.min()), float(x.max()), nb)
        fast, gen = TestFastPath._both(t, ts)
        want = np.append(*oracle.histogram(x, ts.taus))
        assert np.array_equal(fast[0], want) and np.array_equal(gen[0], want)

    def test_hot_bin_and_ties(self, rng):
        """few distinct values: every voxel lands in a handful of bins (atomic
        hot spots, most neighbour pairs tie)."""
        x = rng.integers(0, 3, (33, 61, 128)).astype(np.float32)
        t = torch.from_numpy(x).cuda()
        ts = E.ThresholdSet(np.linspace(-0.5, 2.5, 7))
        fast, gen = TestFastPath._both(t, ts)
        want = np.append(*oracle.histogram(x, ts.taus))
        assert np.array_equal(fast[0], want) and np.array_equal(gen[0], want)


class TestSyntheticKinds:
    """The smooth synthetic kinds of SURVEY §8(d) through the rank4 kernel
    (1024 uniform thresholds, W % 128 == 0): gaussian blobs (c = 0 almost
    everywhere, neighbouring rows share ranks -- the hot-counter pattern of
    the deposits) and the radial gradient (ranks tie along shells), at a
    static-partition depth and a dynamic-schedule depth."""

    @pytest.mark.parametrize("kind", ["gaussian-blobs", "radial-gradient"])
    @pytest.mark.parametrize("dims", [(48, 96, 128), (160, 64, 128)])
    def test_bit_exact(self, kind, dims):
        from paper_2510_20271_b200.synthetic import SyntheticSpec, generate_array

        x = generate_array(SyntheticSpec(kind, dims, seed=3))
        g = E.ScalarGrid(torch.from_numpy(x).cuda())
        ts = E.uniform_thresholds(g, 1024)
        got = E.histogram_device(torch.from_numpy(x).cuda(), ts).cpu().numpy().reshape(-1)
        assert np.array_equal(got, np.append(*oracle.histogram(x, ts.taus)))


class TestEdgeRanking:
    """Edge-table ranking (power-of-two bin counts): voxels sitting exactly on
    thresholds, one ulp either side, at the range ends and outside the range."""

    @pytest.mark.parametrize("nb", [256, 1024, 2048])
    def test_values_on_and_around_thresholds(self, rng, nb):
        ts = E.thresholds_from_range(-1.25, 3.5, nb)
        t32 = ts.taus.astype(np.float32)
        pool = np.concatenate([t32, np.nextafter(t32, np.float32(np.inf)), np.nextafter(t32, np.float32(-np.inf)),
                               np.float32([-1e30, -5.0, -1.25, 3.5, 7.0, 1e30, 0.0, -0.0, 1e-40])])
        x = rng.choice(pool, size=(19, 37, 132)).astype(np.float32)
        t = torch.from_numpy(x).cuda()
        _, b = ts.device_table(_lib_dtype_f32(), t.device)
        assert b.lut_edge == 1
        out = TestFastPath._all(t, ts)
        want = np.append(*oracle.histogram(x, ts.taus))
        for name, h in out.items():
            assert np.array_equal(h[0], want), name


def _lib_dtype_f32():
    from paper_2510_20271_b200 import _lib

    return _lib.DTYPE_F32


class TestHostStreaming:
    """ecc_discrete_host: z-chunks copied on a side stream while the previous
    chunk is deposited; bit-exact with the device-resident call."""

    @pytest.mark.parametrize("resident", [None, False])
    @pytest.mark.parametrize("chunk", [1, 2, 7, 36, 64, 1000])
    def test_chunks_equal_device_call(self, rng, chunk, resident):
        x = rng.random((37, 45, 132)).astype(np.float32)
        ts = E.thresholds_from_range(float(x.min()), float(x.max()), 256)
        want_c, want_h = E.ecc_discrete(torch.from_numpy(x).cuda(), ts, return_hist=True)
        for host in (torch.from_numpy(x), torch.from_numpy(x).pin_memory()):
            for _ in range(2):   # the second call reuses the cached device buffers
                c, h = E.ecc_discrete_host(host, ts, chunk_planes=chunk, return_hist=True, resident=resident)
                assert torch.equal(c, want_c) and torch.equal(h, want_h)

    @pytest.mark.parametrize("resident", [None, False])
    def test_uint8_and_generic_shapes(self, rng, resident):
        x = rng.integers(0, 256, (20, 31, 50), dtype=np.uint8)   # W % 4 != 0: generic kernel
        ts = E.ThresholdSet(np.arange(0.0, 256.0, 9.0))
        c = E.ecc_discrete_host(x, ts, chunk_planes=6, resident=resident)
        assert np.array_equal(c.cpu().numpy(), oracle.curve(x.astype(np.float64), ts.taus))

    def test_single_plane_and_consecutive_volumes(self, rng):
        ts = E.ThresholdSet(np.linspace(0.0, 1.0, 33))
        for dims in ((1, 40, 64), (3, 40, 64), (3, 40, 64)):
            x = torch.from_numpy(rng.random(dims).astype(np.float32)).pin_memory()
            want = E.ecc_discrete(x.cuda(), ts)
            assert torch.equal(E.ecc_discrete_host(x, ts, chunk_planes=2), want)


class TestFastPathU8:
    """uint8 volumes (W % 16 == 0) take the rank kernel with the value as rank."""

    @pytest.mark.parametrize("dims", [(1, 4, 16), (9, 33, 48), (17, 61, 128), (5, 90, 144), (40, 31, 256)])
    def test_u8_volumes(self, rng, dims):
        x = rng.integers(0, 256, dims, dtype=np.uint8)
        t = torch.from_numpy(x).cuda()
        for taus in (np.arange(0.0, 256.0, 1.0), np.arange(2.5, 250.0, 7.25), np.array([-3.0, 0.0, 127.5, 255.0, 300.0])):
            ts = E.ThresholdSet(taus)
            out = TestFastPath._all(t, ts)
            want = np.append(*oracle.histogram(x.astype(np.float64), taus))
            for name, h in out.items():
                assert np.array_equal(h[0], want), (dims, name)

    def test_u8_batched_and_ties(self, rng):
        xs = rng.integers(0, 3, (3, 12, 40, 64), dtype=np.uint8)
        ts = E.ThresholdSet(np.array([0.0, 1.0, 2.0]))
        h = E.histogram_device(torch.from_numpy(xs).cuda(), ts, ndim=3).cpu().numpy()
        for i in range(3):
            assert np.array_equal(h[i], np.append(*oracle.histogram(xs[i].astype(np.float64), ts.taus)))


class TestFastPath2DTiles:
    """2-D grids and D == 1 volumes take the 2-D tile pipeline (float32 and uint8)."""

    @pytest.mark.parametrize("hw", [(4, 16), (30, 128), (31, 132), (61, 260), (200, 48), (1, 64)])
    def test_2d_batches(self, rng, hw):
        xs = rng.random((5,) + hw).astype(np.float32)
        t = torch.from_numpy(xs).cuda()
        for nb in (7, 256, 1024):
            ts = E.thresholds_from_range(float(xs.min()), float(xs.max()), nb)
            out = TestFastPath._all(t, ts, ndim=2)
            for i in range(5):
                want = np.append(*oracle.histogram(xs[i], ts.taus))
                for name, h in out.items():
                    assert np.array_equal(h[i], want), (hw, nb, name, i)

    def test_2d_u8(self, rng):
        xs = rng.integers(0, 256, (4, 70, 128), dtype=np.uint8)
        t = torch.from_numpy(xs).cuda()
        ts = E.ThresholdSet(np.arange(0.0, 256.0, 3.0))
        out = TestFastPath._all(t, ts, ndim=2)
        for i in range(4):
            want = np.append(*oracle.histogram(xs[i].astype(np.float64), ts.taus))
            for name, h in out.items():
                assert np.array_equal(h[i], want), (name, i)


class TestRankTileRows:
    """The rank kernels' y tiling: the first tile of a column deposits lane 0
    (row 0) and the last, bottom-aligned tile deposits lane 31 (row H - 1),
    whose missing neighbours are read from the sentinel row.  Heights on
    both sides of every tiling change (1, 2 or 3 tiles, 30 k + 1, 30 k + 2,
    512), plateau-heavy values so that tie-breaking across the tile
    boundaries matters, f32 (3-D and 2-D kernels) and uint8."""

    HEIGHTS = [2, 31, 32, 33, 34, 61, 62, 63, 64, 91, 92, 93, 94, 122, 152, 512]

    @pytest.mark.parametrize("h", HEIGHTS)
    def test_heights(self, rng, h):
        for dt in (np.float32, np.uint8):
            x = rng.integers(0, 5, (3, h, 144)).astype(dt)
            t = torch.from_numpy(x).cuda()
            ts = E.ThresholdSet(np.array([0.0, 1.0, 2.5, 3.0]))
            want = np.append(*oracle.histogram(x.astype(np.float64), ts.taus))
            out = TestFastPath._all(t, ts)
            for name, hh in out.items():
                assert np.array_equal(hh[0], want), (h, dt, name)
            # the same planes as a batch of 2-D images (the 2-D tile kernel)
            h2 = E.histogram_device(t, ts, ndim=2).cpu().numpy()
            for i in range(3):
                assert np.array_equal(h2[i], np.append(*oracle.histogram(x[i].astype(np.float64), ts.taus))), (h, dt, i)

    def test_uniform_thresholds_512_rows(self, rng):
        """The bench's edge-ranking table (1024 uniform thresholds) on a
        512-row volume: 17 tiles per column instead of 18."""
        x = rng.random((6, 512, 128)).astype(np.float32)
        x[:, ::7, :] = np.round(x[:, ::7, :] * 16) / 16
        t = torch.from_numpy(x).cuda()
        ts = E.thresholds_from_range(float(x.min()), float(x.max()), 1024)
        fast, gen = TestFastPath._both(t, ts)
        assert np.array_equal(fast, gen)
        assert np.array_equal(fast[0], np.append(*oracle.histogram(x, ts.taus)))

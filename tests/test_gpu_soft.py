"""Soft ECC on the GPU against the reference (golden vectors) and the oracle.

Tolerance (north star: 1e-4 relative, fp32): normwise, i.e.
max|gpu - ref| / max|ref| <= 1e-4, for chi, d_tau, d_u, d_values; d_alpha
against the reference's 4th-order finite difference of _forward_raw
(soft.py:308-315) with the gradient_check floor (soft.py:303-306).
Coefficients of the effective field must match the reference exactly.
Mirrors tests/test_soft.py of the reference.
"""

import numpy as np
import pytest
import torch

from conftest import golden_cases, normwise
from oracle import oracle

pytestmark = pytest.mark.gpu

E = pytest.importorskip("paper_2510_20271_b200")

TOL = 1e-4


def _params(golden, k):
    alpha, lam = golden[f"soft{k}_params"]
    return E.SoftEccParams(lam=float(lam), alpha=float(alpha), u=golden[f"soft{k}_u"],
                           taus=E.ThresholdSet(golden[f"soft{k}_taus"]))


class TestGoldenParity:
    def test_effective_field_bit_exact(self, golden):
        for k in golden_cases(golden, "soft"):
            x = golden[f"soft{k}_x"]
            alpha, _ = golden[f"soft{k}_params"]
            eff = E.effective_field(E.ScalarGrid(x), float(alpha), golden[f"soft{k}_u"]).values
            assert np.array_equal(eff, golden[f"soft{k}_eff"]), k

    def test_effective_field_coefficients_exact(self, golden):
        for k in golden_cases(golden, "soft"):
            x = golden[f"soft{k}_x"]
            alpha, lam = golden[f"soft{k}_params"]
            taus = golden[f"soft{k}_taus"]
            p = E.soft._params(float(lam), float(alpha), golden[f"soft{k}_u"], taus[0], taus[-1], x.ndim)
            t = torch.from_numpy(x).cuda()
            c, _ = E.soft.soft_prepare_device(t, x.shape, 1, p)
            assert np.array_equal(c.cpu().numpy(), golden[f"soft{k}_coeffs"]), k

    def test_forward(self, golden):
        for k in golden_cases(golden, "soft"):
            g = E.ScalarGrid(golden[f"soft{k}_x"])
            cg = E.CoefficientGrid(golden[f"soft{k}_coeffs"])
            chi = E.soft_ecc(g, cg, _params(golden, k)).values
            assert chi.dtype == np.float64
            err = normwise(chi, golden[f"soft{k}_chi"])
            assert err <= TOL, (k, err)

    def test_backward(self, golden):
        for k in golden_cases(golden, "soft"):
            g = E.ScalarGrid(golden[f"soft{k}_x"])
            cg = E.CoefficientGrid(golden[f"soft{k}_coeffs"])
            params = _params(golden, k)
            gr = E.soft_ecc_backward(g, cg, params, golden[f"soft{k}_upstream"])
            for name, got in (("dvalues", gr.d_values), ("dtau", gr.d_tau), ("du", gr.d_u)):
                want = golden[f"soft{k}_{name}"]
                if np.abs(want).max() == 0:
                    assert np.abs(got).max() <= 1e-12, (k, name)
                    continue
                err = normwise(got, want)
                assert err <= TOL, (k, name, err)
            assert abs(gr.d_u @ params.u) <= 1e-8
            fd = float(golden[f"soft{k}_dalpha_fd"][0])
            rel = abs(gr.d_alpha - fd) / max(abs(gr.d_alpha), abs(fd), 1e-4)
            assert rel <= TOL, (k, gr.d_alpha, fd)

    def test_closed_forms(self):
        """test_soft.py:39-50, 160-174."""
        g = E.ScalarGrid([[0.0]])
        c = E.compute_coefficients(g)
        u = E.reparametrize_direction([1.0, 0.0])
        for lam in (0.5, 4.0, 100.0):
            p = E.SoftEccParams(lam=lam, alpha=0.0, u=u, taus=E.ThresholdSet([0.0]))
            assert abs(E.soft_ecc(g, c, p).values[0] - 0.5) <= 1e-6
        p = E.SoftEccParams(lam=100.0, alpha=0.0, u=u, taus=E.ThresholdSet([1.0]))
        assert abs(E.soft_ecc(g, c, p).values[0] - 1.0) <= 1e-6
        p = E.SoftEccParams(lam=4.0, alpha=0.0, u=u, taus=E.ThresholdSet([0.0]))
        gr = E.soft_ecc_backward(g, c, p, np.ones(1))
        assert abs(gr.d_tau[0] - 1.0) <= 1e-6 and abs(gr.d_values.ravel()[0] + 1.0) <= 1e-6

    def test_alpha_zero_kills_direction_gradient(self, rng):
        x = rng.integers(0, 10, (6, 7)).astype(np.float64)
        g = E.ScalarGrid(x)
        c = E.compute_coefficients(g)
        p = E.SoftEccParams(lam=3.0, alpha=0.0, u=E.reparametrize_direction([3.0, 4.0]),
                            taus=E.uniform_thresholds(g, 5))
        gr = E.soft_ecc_backward(g, c, p, rng.normal(size=5))
        assert np.array_equal(gr.d_u, np.zeros(2))

    def test_upstream_length_checked(self, rng):
        g = E.ScalarGrid(rng.integers(0, 10, (4, 4)).astype(np.float64))
        p = E.SoftEccParams(lam=1.0, alpha=0.0, u=np.array([1.0, 0.0]), taus=E.uniform_thresholds(g, 4))
        with pytest.raises(ValueError):
            E.soft_ecc_backward(g, E.compute_coefficients(g), p, np.ones(3))


def _oracle_case(rng, dims, B, lam, alpha, u):
    x = rng.random(dims).astype(np.float32).astype(np.float64)
    eff = oracle.effective_field(x, alpha, u)
    c = oracle.coefficients(eff)
    taus = E.uniform_thresholds(E.ScalarGrid(eff), B).taus
    return x, c, taus


class TestOracleParity:
    @pytest.mark.parametrize("dims,B,lam", [((128, 96), 256, 50.0), ((24, 20, 16), 256, 50.0),
                                           ((97, 83), 256, 50.0), ((19, 23, 17), 256, 50.0),   # band kernel, n % 16 != 0
                                           ((64, 64), 1024, 50.0), ((40, 40), 37, 1e4), ((50, 30), 7, 0.5)])
    def test_forward_backward(self, rng, dims, B, lam):
        alpha = 0.3
        u = E.reparametrize_direction([1.0, 2.0, -0.5][: len(dims)])
        x, c, taus = _oracle_case(rng, dims, B, lam, alpha, u)
        params = E.SoftEccParams(lam=lam, alpha=alpha, u=u, taus=E.ThresholdSet(taus))
        g, cg = E.ScalarGrid(x), E.CoefficientGrid(c)
        chi = E.soft_ecc(g, cg, params).values
        want = oracle.soft_forward(x, c, lam, alpha, u, taus)
        assert normwise(chi, want) <= TOL
        up = rng.uniform(0.5, 1.5, taus.size)
        gr = E.soft_ecc_backward(g, cg, params, up)
        dv, dt, du, da, _ = oracle.soft_backward(x, c, lam, alpha, u, taus, up)
        assert normwise(gr.d_values, dv) <= TOL
        assert normwise(gr.d_tau, dt) <= TOL
        assert normwise(gr.d_u, du) <= TOL
        assert abs(gr.d_alpha - da) <= TOL * max(abs(da), 1e-4)

    def test_determinism(self, rng):
        """Bit-identical repeated runs (test_soft.py:296-306)."""
        x = rng.random((96, 96))
        g = E.ScalarGrid(x)
        c = E.compute_coefficients(g)
        p = E.SoftEccParams(lam=8.0, alpha=0.2, u=E.reparametrize_direction([2.0, -1.0]),
                            taus=E.uniform_thresholds(g, 32))
        a = E.soft_ecc(g, c, p).values
        b = E.soft_ecc(g, c, p).values
        assert a.tobytes() == b.tobytes()


def _module_outputs(m, x, up):
    xs = x.clone().requires_grad_(True)
    m.zero_grad()
    chi = m(xs)
    (chi * up).sum().backward()
    return [chi.detach().cpu().numpy(), xs.grad.cpu().numpy(), m.taus.grad.cpu().numpy(), m.v.grad.cpu().numpy(),
            m.alpha.grad.cpu().numpy()]


class TestBandKernel:
    """The windowed soft kernels (ecc_soft.cu band mode: a 128-threshold window
    per voxel, saturated pairs taken as sigma = 0 / 1 with error < 2^-24)
    against the full kernels: same outputs to float32 rounding, over odd
    sizes (direct loads instead of the staged cp.async slices), several
    chunks per CTA, 2-D and 3-D."""

    @pytest.mark.parametrize("shape,v", [((3, 97, 83), [1.0, 2.0]), ((6, 128, 160), [1.0, 2.0]),
                                         ((2, 33, 31, 29), [1.0, 2.0, -0.5]), ((1, 64, 64, 64), [1.0, 2.0, -0.5])])
    @pytest.mark.parametrize("g", [0, 1, 3])
    def test_matches_full_kernels(self, rng, shape, v, g):
        from paper_2510_20271_b200 import _lib

        B, lam, alpha = 256, 50.0, 0.3
        u = np.asarray(v) / np.linalg.norm(v)
        span = alpha * np.abs(u).sum()
        taus = np.linspace(-span, 1.0 + span, B + 1)[1:]
        m = E.SoftECC(taus, v, alpha=alpha, lam=lam).cuda()
        x = torch.from_numpy(rng.random(shape).astype(np.float32)).cuda()
        up = torch.from_numpy(rng.uniform(0.5, 1.5, (shape[0], B))).cuda()
        with _lib.variant(soft_band=0, soft_g=g):
            full = _module_outputs(m, x, up)
        with _lib.variant(soft_band=1, soft_g=g):
            band = _module_outputs(m, x, up)
        for name, a, b in zip(("chi", "dX", "dtau", "dv"), band, full):
            assert normwise(a, b) <= (1e-4 if name == "dv" else 1e-5), name
        assert abs(float(band[4]) - float(full[4])) <= 1e-4 * max(abs(float(full[4])), 1e-3)

    @pytest.mark.parametrize("B", [200, 250, 368])
    def test_threshold_counts(self, rng, B):
        """Partial last blocks and the largest band count (16 bands)."""
        from paper_2510_20271_b200 import _lib
        from paper_2510_20271_b200.soft import band_window

        lam, alpha, v = 50.0 * B / 256, 0.3, [1.0, 2.0]
        u = np.asarray(v) / np.linalg.norm(v)
        span = alpha * np.abs(u).sum()
        taus = np.linspace(-span, 1.0 + span, B + 1)[1:]
        assert band_window(taus, lam) == 128
        m = E.SoftECC(taus, v, alpha=alpha, lam=lam).cuda()
        x = torch.from_numpy(rng.random((2, 64, 72)).astype(np.float32)).cuda()
        up = torch.from_numpy(rng.uniform(0.5, 1.5, (2, B))).cuda()
        with _lib.variant(soft_band=0):
            full = _module_outputs(m, x, up)
        band = _module_outputs(m, x, up)
        # d_v comes from G = sum of -dX pos, a cancelling float32 sum in both
        # kernels (summed in different orders): 1e-4 as against the oracle
        for name, a, b in zip(("chi", "dX", "dtau", "dv"), band, full):
            assert normwise(a, b) <= (1e-4 if name == "dv" else 1e-5), name

    @pytest.mark.parametrize("shape,v", [((3, 97, 83), [1.0, 2.0]), ((2, 33, 31, 29), [1.0, 2.0, -0.5])])
    def test_records_reuse_bit_identical(self, rng, shape, v):
        """The backward that reads the forward's band-sorted records and the one
        that compacts and sorts again see the same records in the same order,
        so d_values, d_tau and G agree bit for bit."""
        B, lam, alpha = 256, 50.0, 0.3
        u = np.asarray(v) / np.linalg.norm(v)
        span = alpha * np.abs(u).sum()
        taus = torch.from_numpy(np.linspace(-span, 1.0 + span, B + 1)[1:]).cuda()
        x = torch.from_numpy(rng.random(shape).astype(np.float32)).cuda()
        ud = torch.from_numpy(u).cuda()
        al = torch.tensor(alpha, dtype=torch.float64, device="cuda")
        nd = len(shape) - 1
        chi, c, fc, lo, params, recs = torch.ops.ecc_b200.soft_ecc_fwd(x, taus, ud, al, lam, nd, True)
        assert recs.numel() > 0
        chi0 = torch.ops.ecc_b200.soft_ecc_fwd(x, taus, ud, al, lam, nd, False)[0]
        assert torch.equal(chi, chi0)   # keeping the records does not change the forward
        up = torch.from_numpy(rng.uniform(0.5, 1.5, (shape[0], B))).cuda()
        with_recs = torch.ops.ecc_b200.soft_ecc_bwd(c, fc, lo, params, taus, up, nd, recs)
        resorted = torch.ops.ecc_b200.soft_ecc_bwd(c, fc, lo, params, taus, up, nd, None)
        for a, b in zip(with_recs, resorted):
            assert torch.equal(a, b)

    def test_records_memory_cap(self, rng, monkeypatch):
        """Above the records memory cap the module keeps no records and the
        backward re-sorts: the same gradients, bit for bit."""
        from paper_2510_20271_b200.soft import SoftECCFunction

        B, v = 256, [1.0, 2.0]
        u = np.asarray(v) / np.linalg.norm(v)
        span = 0.3 * np.abs(u).sum()
        m = E.SoftECC(np.linspace(-span, 1.0 + span, B + 1)[1:], v, alpha=0.3, lam=50.0).cuda()
        x = torch.from_numpy(rng.random((2, 96, 80)).astype(np.float32)).cuda()
        up = torch.from_numpy(rng.uniform(0.5, 1.5, (2, B))).cuda()
        kept = _module_outputs(m, x, up)
        monkeypatch.setattr(SoftECCFunction, "RECORDS_MEMORY_FRACTION", 0.0)
        resorted = _module_outputs(m, x, up)
        for a, b in zip(kept, resorted):
            assert np.array_equal(a, b)

    def test_unsorted_thresholds_fall_back(self, rng):
        """Learnable thresholds may leave sorted order: the band kernels then
        step aside and the full ones run (band_ok)."""
        B, lam, alpha = 256, 50.0, 0.3
        v = np.array([1.0, 2.0])
        u = v / np.linalg.norm(v)
        taus = np.linspace(-0.5, 1.5, B)
        perm = rng.permutation(B)
        m = E.SoftECC(taus[perm], v, alpha=alpha, lam=lam).cuda()
        x = rng.random((2, 48, 40)).astype(np.float32)
        chi = m(torch.from_numpy(x).cuda()).detach().cpu().numpy()
        for i in range(2):
            xi = x[i].astype(np.float64)
            c = oracle.coefficients(oracle.effective_field(xi, alpha, u))
            assert normwise(chi[i], oracle.soft_forward(xi, c, lam, alpha, u, taus[perm])) <= TOL


class TestModule:
    def test_module_gradients_vs_oracle(self, rng):
        N, H, W, B = 3, 40, 36, 64
        x = rng.random((N, H, W)).astype(np.float32)
        v = np.array([1.0, 2.0])
        alpha, lam = 0.3, 50.0
        u = v / np.linalg.norm(v)
        taus0 = np.linspace(-0.4, 1.4, B)
        m = E.SoftECC(taus0, v, alpha=alpha, lam=lam).cuda()
        xt = torch.from_numpy(x).cuda().requires_grad_(True)
        chi = m(xt)
        assert chi.shape == (N, B)
        up = torch.from_numpy(rng.uniform(0.5, 1.5, (N, B))).cuda()
        (chi * up).sum().backward()
        gtau = np.zeros(B)
        G = np.zeros(2)
        for i in range(N):
            xi = x[i].astype(np.float64)
            c = oracle.coefficients(oracle.effective_field(xi, alpha, u))
            want = oracle.soft_forward(xi, c, lam, alpha, u, taus0)
            assert normwise(chi[i].detach().cpu().numpy(), want) <= TOL
            dv, dt, _, _, Gi = oracle.soft_backward(xi, c, lam, alpha, u, taus0, up[i].cpu().numpy())
            assert normwise(xt.grad[i].cpu().numpy(), dv) <= TOL
            gtau += dt
            G += Gi
        assert normwise(m.taus.grad.cpu().numpy(), gtau) <= TOL
        # u = v/|v|: dL/dv = jvp^T(-alpha G) ; dL/dalpha = -G.u
        du_raw = -alpha * G
        dv_want = (du_raw - u * (u @ du_raw)) / np.linalg.norm(v)
        assert normwise(m.v.grad.cpu().numpy(), dv_want) <= TOL
        da = -(G @ u)
        assert abs(float(m.alpha.grad) - da) <= TOL * max(abs(da), 1e-4)

    def test_module_3d_batch(self, rng):
        x = torch.from_numpy(rng.random((2, 12, 10, 9)).astype(np.float32)).cuda()
        m = E.SoftECC(np.linspace(0, 1, 16), [1.0, 2.0, -0.5], alpha=0.25, lam=10.0).cuda()
        chi = m(x)
        assert chi.shape == (2, 16)
        chi.sum().backward()
        assert m.taus.grad is not None and m.v.grad is not None and m.alpha.grad is not None


class TestModule3D:
    def test_3d_batch_vs_oracle(self, rng):
        N, D, H, W, B = 2, 10, 12, 9, 40
        x = rng.random((N, D, H, W)).astype(np.float32)
        v = np.array([1.0, 2.0, -0.5])
        u = v / np.linalg.norm(v)
        alpha, lam = 0.25, 20.0
        taus0 = np.linspace(-0.4, 1.4, B)
        m = E.SoftECC(taus0, v, alpha=alpha, lam=lam).cuda()
        xt = torch.from_numpy(x).cuda().requires_grad_(True)
        chi = m(xt)
        up = torch.from_numpy(rng.uniform(0.5, 1.5, (N, B))).cuda()
        (chi * up).sum().backward()
        gtau = np.zeros(B)
        G = np.zeros(3)
        for i in range(N):
            xi = x[i].astype(np.float64)
            c = oracle.coefficients(oracle.effective_field(xi, alpha, u))
            assert normwise(chi[i].detach().cpu().numpy(), oracle.soft_forward(xi, c, lam, alpha, u, taus0)) <= TOL
            dv, dt, _, _, Gi = oracle.soft_backward(xi, c, lam, alpha, u, taus0, up[i].cpu().numpy())
            assert normwise(xt.grad[i].cpu().numpy(), dv) <= TOL
            gtau += dt
            G += Gi
        assert normwise(m.taus.grad.cpu().numpy(), gtau) <= TOL
        da = -(G @ u)
        assert abs(float(m.alpha.grad) - da) <= TOL * max(abs(da), 1e-4)

    def test_sharp_lambda_direct_mode_module(self, rng):
        """lam * threshold spread too large for the factorised sigmoid: float64-exponent mode."""
        x = rng.random((24, 20)).astype(np.float32)
        taus0 = np.linspace(0.0, 1.0, 16)
        m = E.SoftECC(taus0, [1.0, 0.0], alpha=0.0, lam=2000.0).cuda()
        xt = torch.from_numpy(x).cuda().requires_grad_(True)
        chi = m(xt)
        chi.sum().backward()
        xi = x.astype(np.float64)
        c = oracle.coefficients(xi)
        assert normwise(chi.detach().cpu().numpy(), oracle.soft_forward(xi, c, 2000.0, 0.0, [1.0, 0.0], taus0)) <= TOL
        dv, dt, _, _, _ = oracle.soft_backward(xi, c, 2000.0, 0.0, [1.0, 0.0], taus0, np.ones(16))
        assert normwise(xt.grad.cpu().numpy(), dv) <= TOL
        assert normwise(m.taus.grad.cpu().numpy(), dt) <= TOL


@pytest.mark.gpu
class TestGradientCheck:
    """gradient_check (soft.py:260-359) on the device: float64 4th-order finite
    differences against the fp32 analytic kernels."""

    def _case(self, rng, dims, ndim_u, lam, nb, alpha=0.3):
        x = rng.random(dims).astype(np.float32).astype(np.float64)
        u = E.reparametrize_direction([1.0, 2.0, -0.5][:ndim_u])
        f = oracle.effective_field(x, alpha, u)
        taus = np.unique(np.linspace(f.min(), f.max(), nb))
        return x, E.SoftEccParams(lam=lam, alpha=alpha, u=u, taus=E.ThresholdSet(taus))

    def test_fd_harness_matches_oracle_gradients(self, rng):
        """The FD harness differentiates the reference's loss: its result equals
        the oracle's float64 analytic gradients to truncation error."""
        for dims, k, lam, nb in [((24, 20), 2, 50.0, 64), ((7, 8, 9), 3, 10.0, 32)]:
            x, params = self._case(rng, dims, k, lam, nb)
            rep = E.gradient_check(E.ScalarGrid(x), params)
            for key in ("d_values", "d_tau", "d_u", "d_alpha"):
                assert rep["normwise"][key] <= 1e-4, (dims, key, rep)
            assert rep["tangency"] <= 1e-8
            # the harness itself against the oracle (float64 analytic)
            up = np.random.default_rng(0).uniform(0.5, 1.5, size=len(params.taus))
            c = oracle.coefficients(oracle.effective_field(x, params.alpha, params.u))
            dv, dt, du, da, _ = oracle.soft_backward(x, c, params.lam, params.alpha, params.u, params.taus.taus, up)
            g = E.soft_ecc_backward(E.ScalarGrid(x), E.CoefficientGrid(c), params, up)
            assert normwise(g.d_tau, dt) <= 1e-4 and normwise(g.d_values, dv) <= 1e-4

    def test_dalpha_against_reference_fd(self, golden):
        """the harness's d_alpha equals the reference's own FD of _forward_raw in alpha (golden)."""
        n = int(golden["manifest"][2])
        checked = 0
        for k in range(n):
            x = golden[f"soft{k}_x"]
            alpha, lam = (float(v) for v in golden[f"soft{k}_params"])
            if x.size < 16 or alpha == 0.0:
                continue
            u = golden[f"soft{k}_u"]
            params = E.SoftEccParams(lam=lam, alpha=alpha, u=u, taus=E.ThresholdSet(golden[f"soft{k}_taus"]))
            rep = E.gradient_check(E.ScalarGrid(x), params, upstream=golden[f"soft{k}_upstream"])
            want = float(golden[f"soft{k}_dalpha_fd"][0])
            assert abs(rep["fd_alpha"] - want) <= 1e-6 * max(1.0, abs(want)), (k, rep["fd_alpha"], want)
            assert rep["normwise"]["d_alpha"] <= 1e-4, (k, rep)
            checked += 1
        assert checked >= 3

    def test_realistic_size(self, rng):
        """256 x 256, 256 thresholds, lambda = 50: far beyond the reference's
        per-pixel loop, every gradient within 1e-4 normwise."""
        x, params = self._case(rng, (256, 256), 2, 50.0, 256)
        rep = E.gradient_check(E.ScalarGrid(x), params)
        for key in ("d_values", "d_tau", "d_u", "d_alpha"):
            assert rep["normwise"][key] <= 1e-4, (key, rep)
        assert rep["tangency"] <= 1e-8


class TestPrepare2D:
    """The 2-D soft prepare kernel (soft_prep2d_kernel) against the generic
    sweep: the same coefficients and centred field, bit for bit."""

    @pytest.mark.parametrize("hw,batch", [((8, 8), 1), ((37, 23), 2), ((70, 33), 3), ((1, 40), 2), ((65, 1), 1),
                                          ((100, 130), 2)])
    def test_matches_generic_sweep(self, rng, hw, batch):
        for dtype, lam, hw_, alpha in ((np.float32, 50.0, 0.01, 0.3), (np.float64, 500.0, 1.0, 0.3),
                                       (np.float32, 50.0, 0.01, 0.0)):
            x = rng.random((batch,) + hw).astype(dtype)
            x[..., ::3, :] = np.round(x[..., ::3, :] * 4) / 4       # ties in the effective field
            u = E.reparametrize_direction([1.0, 2.0])
            p = E.soft._params(lam, alpha, u, -0.5, 1.5, 2, hw_)
            t = torch.from_numpy(x).cuda()
            c1, (f1, l1) = E.soft.soft_prepare_device(t, hw, batch, p)
            with E._lib.variant(generic=1):
                c2, (f2, l2) = E.soft.soft_prepare_device(t, hw, batch, p)
            assert torch.equal(c1, c2) and torch.equal(f1, f2), (hw, dtype, alpha)
            if l1 is not None:
                assert torch.equal(l1, l2)
            with E._lib.variant(soft_prep=1):   # the per-voxel tile kernel
                c3, (f3, _) = E.soft.soft_prepare_device(t, hw, batch, p)
            assert torch.equal(c1, c3) and torch.equal(f1, f3), (hw, dtype, alpha)
            xi = x[0].astype(np.float64)
            want = oracle.coefficients(oracle.effective_field(xi, alpha, u))
            assert np.array_equal(c1[0].cpu().numpy(), want), (hw, dtype, alpha)

    def test_nonfinite_tiles_fall_back(self, rng):
        hw = (70, 90)
        x = rng.random((2,) + hw).astype(np.float32)
        x[0, 5, 7] = np.nan
        x[1, 69, 89] = np.inf
        x[1, 0, 30] = -np.inf
        u = E.reparametrize_direction([1.0, 2.0])
        p = E.soft._params(50.0, 0.3, u, -0.5, 1.5, 2, 0.01)
        t = torch.from_numpy(x).cuda()
        c1, (f1, _) = E.soft.soft_prepare_device(t, hw, 2, p)
        with E._lib.variant(generic=1):
            c2, (f2, _) = E.soft.soft_prepare_device(t, hw, 2, p)
        assert torch.equal(c1, c2)
        assert torch.equal(f1.view(torch.int32), f2.view(torch.int32))


class TestPrepare3D:
    """The dedicated 3-D soft prepare (soft_prep3d_kernel) against the generic
    sweep: the same coefficients of the effective field and the same centred
    field and remainder, bit for bit (float32 and float64 grids, ragged
    shapes, ties, with and without the position term)."""

    @pytest.mark.parametrize("dhw,batch", [((5, 6, 7), 1), ((17, 33, 40), 2), ((9, 1, 35), 1), ((1, 20, 64), 2),
                                           ((40, 18, 31), 1)])
    def test_matches_generic_sweep(self, rng, dhw, batch):
        for dtype, lam, hw_, alpha in ((np.float32, 50.0, 0.01, 0.3), (np.float64, 500.0, 1.0, 0.25),
                                       (np.float32, 50.0, 0.01, 0.0)):
            x = rng.random((batch,) + dhw).astype(dtype)
            x[..., ::2, :, :] = np.round(x[..., ::2, :, :] * 4) / 4       # ties in the effective field
            u = E.reparametrize_direction([1.0, 2.0, -0.5])
            p = E.soft._params(lam, alpha, u, -0.5, 1.5, 3, hw_)
            t = torch.from_numpy(x).cuda()
            c1, (f1, l1) = E.soft.soft_prepare_device(t, dhw, batch, p)
            with E._lib.variant(generic=1):
                c2, (f2, l2) = E.soft.soft_prepare_device(t, dhw, batch, p)
            assert torch.equal(c1, c2) and torch.equal(f1, f2), (dhw, dtype, alpha)
            if l1 is not None:
                assert torch.equal(l1, l2)
            # and the coefficients against the oracle's of the float64 field
            xi = x[0].astype(np.float64)
            want = oracle.coefficients(oracle.effective_field(xi, alpha, u))
            assert np.array_equal(c1[0].cpu().numpy(), want), (dhw, dtype, alpha)

    @pytest.mark.parametrize("dhw", [(33, 64, 70), (64, 61, 96), (9, 95, 33)])
    def test_row_word_kernel_vs_tile_kernel(self, rng, dhw):
        """The row-word prepare (default) against the per-voxel tile kernel
        (soft_prep=1) on several tiles, chunks and ragged edges, with ties."""
        u = E.reparametrize_direction([1.0, 2.0, -0.5])
        for dtype, alpha in ((np.float32, 0.3), (np.float64, 0.25), (np.float32, 0.0)):
            x = rng.random((2,) + dhw).astype(dtype)
            x[:, :, ::3, :] = np.round(x[:, :, ::3, :] * 8) / 8
            p = E.soft._params(50.0, alpha, u, -0.5, 1.5, 3, 0.01)
            t = torch.from_numpy(x).cuda()
            c1, (f1, _) = E.soft.soft_prepare_device(t, dhw, 2, p)
            with E._lib.variant(soft_prep=1):
                c2, (f2, _) = E.soft.soft_prepare_device(t, dhw, 2, p)
            assert torch.equal(c1, c2) and torch.equal(f1, f2), (dhw, dtype, alpha)

    def test_nonfinite_tiles_fall_back(self, rng):
        """A non-finite effective field: the tile is redone with the IEEE
        compares, matching the generic sweep bit for bit."""
        dhw = (12, 40, 70)
        x = rng.random((1,) + dhw).astype(np.float32)
        x[0, 5, 7, 9] = np.nan
        x[0, 11, 39, 69] = np.inf
        x[0, 0, 0, 40] = -np.inf
        u = E.reparametrize_direction([1.0, 2.0, -0.5])
        p = E.soft._params(50.0, 0.3, u, -0.5, 1.5, 3, 0.01)
        t = torch.from_numpy(x).cuda()
        c1, (f1, _) = E.soft.soft_prepare_device(t, dhw, 1, p)
        with E._lib.variant(generic=1):
            c2, (f2, _) = E.soft.soft_prepare_device(t, dhw, 1, p)
        assert torch.equal(c1, c2)
        assert torch.equal(f1.view(torch.int32), f2.view(torch.int32))

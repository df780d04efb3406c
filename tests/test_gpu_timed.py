"""Parity at the benchmarked sizes (VERDICT r1 "what's missing" #1).

Every configuration bench.py times is checked here against the CPU oracle on
the same inputs, not only through size-independent invariants:

* C2  -- 512^3 float32 counter volume, 1024 uniform thresholds (bench seed):
  bit-exact histogram, overflow and curve.
* NS  -- 1024^3, the north-star volume: bit-exact, the oracle accumulated
  slab by slab (oracle/parity.py) so the host never holds the volume.
* C5  -- 256-plane slabs of 2048 x 2048 planes through ecc_histogram_range
  (the per-rank call of distributed.slab_histogram), summed over a partition.
* C3  -- full 1024 x 1024 images, B = 256, lambda = 50, alpha = 0.3, through
  the SoftECC module: chi, d_values, d_tau, d_v, d_alpha normwise <= 1e-4.
* C4  -- a 128^3 volume through the same 3-D module path.

The reference's harness refuses to report a time for a wrong answer
(/root/reference/pkg/src/ecckit/bench.py:28-37, 115-117); bench.py applies
the same gate per leg with these helpers.
"""

import numpy as np
import pytest
import torch

from conftest import normwise
from oracle import oracle, parity

pytestmark = pytest.mark.gpu

E = pytest.importorskip("paper_2510_20271_b200")
from paper_2510_20271_b200 import _lib  # noqa: E402

import bench  # noqa: E402  (the bench's seeds and sizes: the test checks exactly what is timed)

TOL = 1e-4
NB = bench.NB


def _counter_device(seed, shape, start=0):
    x = torch.empty(shape, dtype=torch.float32, device="cuda")
    _lib.check(_lib.lib().ecc_counter_grid(seed, start, x.numel(), _lib.ptr(x), _lib.stream_ptr(x)))
    return x


def _hist_device(x, taus):
    return E.histogram_device(x, taus).cpu().numpy().reshape(-1)


def test_c2_512_cubed_bit_exact():
    n = 512
    x = _counter_device(bench.SEED, (n, n, n))
    lo, hi, nonfinite = E.device_minmax(x)
    assert nonfinite == 0
    taus = E.thresholds_from_range(lo, hi, NB)
    got = _hist_device(x, taus)
    want = parity.counter_slab_hist(bench.SEED, (n, n, n), 0, n, taus.taus)
    assert np.array_equal(got, want)
    curve = E.ecc_discrete(x, taus).cpu().numpy().reshape(-1)
    assert curve.dtype == np.int64
    assert np.array_equal(curve, np.cumsum(want[:-1]))
    # the same volume through the reference-shaped API on a host array
    host = x.cpu().numpy()
    assert np.array_equal(E.compute_ecc(E.ScalarGrid(host), taus).values, np.cumsum(want[:-1]))


def test_ns_1024_cubed_bit_exact():
    n = 1024
    x = _counter_device(bench.SEED + 1, (n, n, n))
    lo, hi, _ = E.device_minmax(x)
    taus = E.thresholds_from_range(lo, hi, NB)
    got = _hist_device(x, taus)
    del x
    torch.cuda.empty_cache()
    want = parity.counter_slab_hist(bench.SEED + 1, (n, n, n), 0, n, taus.taus, slab=128)
    assert np.array_equal(got, want)
    assert int(got.sum()) == 1


def test_c5_slabs_bit_exact():
    """C5's per-rank call (bench_c5_slab, distributed.slab_histogram): two
    256-plane z-slabs of 2048 x 2048 planes, each swept by
    ecc_histogram_range over its own planes with the neighbour's halo plane,
    summed as the NCCL all-reduce sums them.  The sum is bit-exact with the
    reference's histogram of the 512 planes.  (A single slab's partial
    histogram follows the kernel's rank order, in which a cell whose two
    highest vertices share a bin may be counted by the other slab; only the
    sum over a partition is order-independent -- DESIGN.md section 5.)"""
    P, H, W = 256, 2048, 2048
    seed = bench.SEED + 2
    taus = E.thresholds_from_range(0.0, 1.0 - 2.0 ** -24, NB)
    got = np.zeros(NB + 1, dtype=np.int64)
    for z0, first, nplanes in ((0, 0, P + 1), (P, P - 1, P + 1)):
        view = _counter_device(seed, (nplanes, H, W), start=first * H * W)
        table, binning = taus.device_table(_lib.DTYPE_F32, view.device)
        dims = _lib.dims_arg(view.shape)
        zlo = z0 - first
        part = torch.empty(NB + 1, dtype=torch.int64, device="cuda")
        _lib.check(_lib.lib().ecc_histogram_range(_lib.ptr(view), _lib.DTYPE_F32, 3, _lib.ptr(dims), 1, zlo, zlo + P,
                                                  _lib.ptr(table), _lib.ctypes.byref(binning), _lib.ptr(part),
                                                  _lib.stream_ptr(view)))
        got += part.cpu().numpy()
        del view
    torch.cuda.empty_cache()
    want = parity.counter_slab_hist(seed, (2 * P, H, W), 0, 2 * P, taus.taus, slab=32)
    assert np.array_equal(got, want)
    assert int(got.sum()) == 1


def _soft_module_case(x_np, taus0, v, alpha, lam, up_np):
    m = E.SoftECC(taus0, v, alpha=alpha, lam=lam).cuda()
    xt = torch.from_numpy(x_np).cuda().requires_grad_(True)
    chi = m(xt)
    (chi * torch.from_numpy(up_np).cuda()).sum().backward()
    return m, xt, chi


@pytest.mark.parametrize("batch", [1, 2])
def test_c3_full_images(batch):
    """C3's configuration on full 1024 x 1024 images (bench_soft: B = 256,
    lambda = 50, alpha = 0.3, u = normalize(1, 2), taus = linspace)."""
    rng = np.random.default_rng(bench.SEED)
    H = W = 1024
    B, lam, alpha = 256, 50.0, 0.3
    v = np.array([1.0, 2.0])
    u = v / np.linalg.norm(v)
    span = alpha * np.abs(u).sum()
    taus0 = np.linspace(-span, 1.0 + span, B + 1)[1:]
    x = rng.random((batch, H, W)).astype(np.float32)
    up = rng.uniform(0.5, 1.5, (batch, B))
    m, xt, chi = _soft_module_case(x, taus0, v, alpha, lam, up)
    gtau, G = np.zeros(B), np.zeros(2)
    for i in range(batch):
        c_chi, dv, dt, _, _, Gi = parity.soft_item(x[i], lam, alpha, u, taus0, up[i])
        assert normwise(chi[i].detach().cpu().numpy(), c_chi) <= TOL
        assert normwise(xt.grad[i].cpu().numpy(), dv) <= TOL
        gtau += dt
        G += Gi
    assert normwise(m.taus.grad.cpu().numpy(), gtau) <= TOL
    du_raw = -alpha * G
    dv_want = (du_raw - u * (u @ du_raw)) / np.linalg.norm(v)
    assert normwise(m.v.grad.cpu().numpy(), dv_want) <= TOL
    da = -(G @ u)
    assert abs(float(m.alpha.grad) - da) <= TOL * max(abs(da), 1e-4)


def test_c4_subvolume_128_cubed():
    """C4's 3-D path (bench_c4: B = 256, lambda = 50, alpha = 0.3,
    u = normalize(1, 2, -0.5)) on a 128^3 volume."""
    rng = np.random.default_rng(bench.SEED + 100)
    n, B, lam, alpha = 128, 256, 50.0, 0.3
    v = np.array([1.0, 2.0, -0.5])
    u = v / np.linalg.norm(v)
    span = alpha * np.abs(u).sum()
    taus0 = np.linspace(-span, 1.0 + span, B + 1)[1:]
    x = rng.random((1, n, n, n)).astype(np.float32)
    up = rng.uniform(0.5, 1.5, (1, B))
    m, xt, chi = _soft_module_case(x, taus0, v, alpha, lam, up)
    c_chi, dv, dt, _, _, G = parity.soft_item(x[0], lam, alpha, u, taus0, up[0])
    assert normwise(chi[0].detach().cpu().numpy(), c_chi) <= TOL
    assert normwise(xt.grad[0].cpu().numpy(), dv) <= TOL
    assert normwise(m.taus.grad.cpu().numpy(), dt) <= TOL
    du_raw = -alpha * G
    dv_want = (du_raw - u * (u @ du_raw)) / np.linalg.norm(v)
    assert normwise(m.v.grad.cpu().numpy(), dv_want) <= TOL
    da = -(G @ u)
    assert abs(float(m.alpha.grad) - da) <= TOL * max(abs(da), 1e-4)

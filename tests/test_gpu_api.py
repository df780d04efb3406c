"""API-level behaviour on the GPU (missing #5-#6):

* NaN / Inf inputs raise ValueError on the torch-native path, as ScalarGrid
  does (/root/reference/pkg/src/ecckit/grid.py:63-64), with the check fused
  into the sweep;
* concurrent calls from two threads on two streams are reentrant and
  bit-exact (the reference's functions are pure);
* SoftECC forward + backward issue no device -> host read, so they capture
  in a CUDA graph, and trace through torch.compile without graph breaks
  (torch.library custom ops with fake implementations);
* a module left on the CPU still computes on the input's device;
* bin counts beyond the shared-memory histogram use the global-memory sweep;
* batch-sharded SoftECC gradients, summed over the shards, equal the full
  batch's (the DDP-style all-reduce of distributed.allreduce_soft_grads).
"""

import threading

import numpy as np
import pytest
import torch

from conftest import normwise
from oracle import oracle

pytestmark = pytest.mark.gpu

E = pytest.importorskip("paper_2510_20271_b200")
from paper_2510_20271_b200 import _lib  # noqa: E402


class TestNonFinite:
    @pytest.mark.parametrize("shape,dtype", [((20, 24, 128), torch.float32),    # rank4, every voxel deposits
                                             ((20, 24, 64), torch.float32),     # rank4 with dummy counters
                                             ((3, 40, 64), torch.float32),      # batched 2-D images (ndim=2)
                                             ((9, 11, 13), torch.float32),      # generic sweep (W % 4 != 0)
                                             ((9, 11, 12), torch.float64)])     # float64 generic sweep
    @pytest.mark.parametrize("bad", [float("nan"), float("inf"), -float("inf")])
    def test_ecc_discrete_rejects(self, rng, shape, dtype, bad):
        x = torch.from_numpy(rng.random(shape)).to("cuda", dtype)
        ndim = 2 if shape == (3, 40, 64) else None
        ts = E.thresholds_from_range(0.0, 1.0, 1024)
        E.ecc_discrete(x, ts, ndim=ndim)    # finite: no error
        idx = tuple(int(rng.integers(0, s)) for s in shape)
        x[idx] = bad
        with pytest.raises(ValueError):
            E.ecc_discrete(x, ts, ndim=ndim)
        # opt-out: no check, no raise (asynchronous path)
        E.ecc_discrete(x, ts, ndim=ndim, check_finite=False)

    def test_last_voxel_and_edge_columns(self, rng):
        ts = E.thresholds_from_range(0.0, 1.0, 1024)
        for idx in [(15, 31, 255), (0, 0, 0), (7, 13, 127), (7, 13, 128), (15, 0, 31)]:
            x = torch.rand((16, 32, 256), device="cuda")
            x[idx] = float("nan")
            with pytest.raises(ValueError):
                E.histogram_device(x, ts, check_finite=True)

    def test_partial_tiles_do_not_report_fill(self, rng):
        """out-of-grid columns carry the TMA's NaN fill; they must not count."""
        ts = E.thresholds_from_range(0.0, 1.0, 1024)
        for shape in [(5, 33, 100), (4, 70, 36), (3, 31, 4)]:
            x = torch.from_numpy(rng.random(shape).astype(np.float32)).cuda()
            h = E.histogram_device(x, ts, check_finite=True).cpu().numpy()[0]
            assert np.array_equal(h, np.append(*oracle.histogram(x.cpu().numpy(), ts.taus))), shape


class TestReentrancy:
    def test_two_threads_two_streams(self, rng):
        vols = [rng.random((96, 64, 128)).astype(np.float32) for _ in range(2)]
        ts = E.thresholds_from_range(0.0, 1.0, 1024)
        want = [np.cumsum(oracle.histogram(v, ts.taus)[0]) for v in vols]
        hosts = [torch.from_numpy(v).pin_memory() for v in vols]
        devs = [torch.from_numpy(v).cuda() for v in vols]
        errors = []

        def worker(i):
            try:
                s = torch.cuda.Stream()
                with torch.cuda.stream(s):
                    for rep in range(6):
                        a = E.ecc_discrete_host(hosts[i], ts, chunk_planes=16).cpu().numpy()
                        b = E.ecc_discrete(devs[i], ts).cpu().numpy()
                        if not (np.array_equal(a, want[i]) and np.array_equal(b, want[i])):
                            errors.append((i, rep))
            except Exception as e:  # noqa: BLE001
                errors.append(repr(e))

        th = [threading.Thread(target=worker, args=(i,)) for i in range(2)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        assert not errors, errors
        E.release_host_buffers()

    def test_many_dynamic_launches_in_flight(self):
        """More dynamic-schedule launches in flight than work-queue slots (64):
        a slot is reused only after its previous launch finished."""
        ts = E.thresholds_from_range(0.0, 1.0, 1024)
        x = torch.rand((256, 128, 128), device="cuda")
        with _lib.variant(zunit=8):
            ref = E.histogram_device(x, ts).clone()
            streams = [torch.cuda.Stream() for _ in range(4)]
            outs = []
            for k in range(96):
                with torch.cuda.stream(streams[k % 4]):
                    outs.append(E.histogram_device(x, ts))
            torch.cuda.synchronize()
        for o in outs:
            assert torch.equal(o, ref)


def _module_case(ndim=2):
    if ndim == 2:
        return E.SoftECC(np.linspace(-0.4, 1.4, 64), [1.0, 2.0], alpha=0.3, lam=50.0).cuda(), (3, 96, 80)
    return E.SoftECC(np.linspace(-0.4, 1.4, 48), [1.0, 2.0, -0.5], alpha=0.25, lam=20.0).cuda(), (2, 20, 24, 16)


class TestSyncFreeModule:
    def test_cuda_graph_capture(self):
        m, shape = _module_case(2)
        x = torch.rand(shape, device="cuda")
        up = torch.rand((shape[0], 64), device="cuda", dtype=torch.float64)

        def step():
            m.zero_grad(set_to_none=False)
            (m(x) * up).sum().backward()
            return m.taus.grad.clone(), m.v.grad.clone(), m.alpha.grad.clone()

        # eager reference (warm-up also allocates the .grad buffers)
        ref = step()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for _ in range(2):
                step()
        torch.cuda.current_stream().wait_stream(s)
        g = torch.cuda.CUDAGraph()
        m.zero_grad(set_to_none=False)
        with torch.cuda.graph(g):
            (m(x) * up).sum().backward()
        x.copy_(x)   # same inputs
        m.zero_grad(set_to_none=False)
        g.replay()
        torch.cuda.synchronize()
        for a, b in zip((m.taus.grad, m.v.grad, m.alpha.grad), ref):
            assert torch.equal(a, b)

    def test_torch_compile_fullgraph(self):
        m, shape = _module_case(3)
        x = torch.rand(shape, device="cuda")
        eager = m(x).detach().clone()
        cm = torch.compile(m, fullgraph=True)
        out = cm(x)
        assert torch.equal(out.detach(), eager)
        out.sum().backward()
        assert m.taus.grad is not None and m.alpha.grad is not None

    def test_module_left_on_cpu(self):
        """taus on the host must not reach a kernel as a device pointer."""
        m = E.SoftECC(np.linspace(0.0, 1.0, 16), [1.0, 2.0], alpha=0.2, lam=10.0)   # not moved to cuda
        x = torch.rand((2, 24, 20), device="cuda")
        ref = E.SoftECC(np.linspace(0.0, 1.0, 16), [1.0, 2.0], alpha=0.2, lam=10.0).cuda()(x)
        assert torch.equal(m(x), ref)
        with pytest.raises(ValueError):
            m(x.cpu())


class TestManyBins:
    def test_float64_beyond_shared_histogram(self, rng):
        x = rng.random((9, 10, 11))
        taus = np.sort(rng.random(40000))
        taus = np.unique(taus)
        ts = E.ThresholdSet(taus)
        h = E.accumulate_histogram(E.ScalarGrid(x), ts)
        want, ovf = oracle.histogram(x, ts.taus)
        assert np.array_equal(h.bins, want) and h.overflow == ovf

    def test_float32_beyond_shared_histogram(self, rng):
        x = rng.random((7, 12, 13)).astype(np.float32)
        ts = E.ThresholdSet(np.unique(np.sort(rng.random(60000))))
        got = E.histogram_device(torch.from_numpy(x).cuda(), ts).cpu().numpy()[0]
        assert np.array_equal(got, np.append(*oracle.histogram(x, ts.taus)))


def test_sharded_gradients_sum_to_full_batch():
    """Batch-sharded SoftECC (distributed.shard_batch): the shared parameters'
    gradients of the shards, summed (what allreduce_soft_grads does), equal
    the full batch's to float64 rounding."""
    from paper_2510_20271_b200 import distributed as D

    x = torch.rand((5, 64, 48), device="cuda")
    taus = np.linspace(-0.4, 1.4, 96)
    full = E.SoftECC(taus, [1.0, 2.0], alpha=0.3, lam=50.0).cuda()
    full(x).sum().backward()
    parts = []
    for r in range(2):
        i0, i1 = D.shard_batch(5, 2, r)
        m = E.SoftECC(taus, [1.0, 2.0], alpha=0.3, lam=50.0).cuda()
        m(x[i0:i1]).sum().backward()
        parts.append(m)
    for name in ("taus", "v", "alpha"):
        a = sum(getattr(p, name).grad for p in parts)
        b = getattr(full, name).grad
        assert normwise(a.cpu().numpy(), b.cpu().numpy()) <= 1e-12, name


def test_soft_step_host_matches_device_batch():
    """soft_step_host (micro-batches copied from pinned host memory while the
    previous one computes) gives the full batch's chi and gradients."""
    x = torch.rand((7, 96, 80))
    up = torch.rand((7, 64), dtype=torch.float64, device="cuda")
    ref = E.SoftECC(np.linspace(-0.4, 1.4, 64), [1.0, 2.0], alpha=0.3, lam=50.0).cuda()
    chi_ref = ref(x.cuda())
    (chi_ref * up).sum().backward()
    m = E.SoftECC(np.linspace(-0.4, 1.4, 64), [1.0, 2.0], alpha=0.3, lam=50.0).cuda()
    chi = E.soft_step_host(m, x.pin_memory(), up, micro=3)
    torch.cuda.synchronize()
    assert normwise(chi.cpu().numpy(), chi_ref.detach().cpu().numpy()) <= 1e-12
    for name in ("taus", "v", "alpha"):
        assert normwise(getattr(m, name).grad.cpu().numpy(), getattr(ref, name).grad.cpu().numpy()) <= 1e-12, name
    with pytest.raises(ValueError):
        E.soft_step_host(m, x.cuda())



@pytest.mark.parametrize("slab,records", [(16, True), (64, True), (16, False)])
def test_soft_step_host_streams_a_3d_item(slab, records, monkeypatch):
    """One 3-D item from host memory is streamed in z-slabs (prepare and
    forward of the resident planes overlap the rest of the copy); chi, the
    coefficients, the fields and every gradient equal the device path's bit
    for bit -- the same kernels over the same voxels, units straddling planes
    included (48 x 64 planes, 4096-voxel chunks)."""
    B = 256
    v = [1.0, 2.0, -0.5]
    u = np.asarray(v) / np.linalg.norm(v)
    span = 0.3 * np.abs(u).sum()
    taus = np.linspace(-span, 1.0 + span, B + 1)[1:]
    x = torch.rand((1, 70, 48, 64), generator=torch.Generator().manual_seed(3))
    up = torch.rand((1, B), dtype=torch.float64, device="cuda") + 0.5
    ref = E.SoftECC(taus, v, alpha=0.3, lam=50.0).cuda()
    chi_ref = ref(x.cuda())
    (chi_ref * up).sum().backward()
    m = E.SoftECC(taus, v, alpha=0.3, lam=50.0).cuda()
    if not records:   # the streamed backward then compacts and sorts itself
        from paper_2510_20271_b200.soft import SoftECCFunction

        monkeypatch.setattr(SoftECCFunction, "RECORDS_MEMORY_FRACTION", 0.0)
    chi = E.soft_step_host(m, x.pin_memory(), up, micro=1, slab_planes=slab)
    torch.cuda.synchronize()
    assert torch.equal(chi, chi_ref.detach())
    for name in ("taus", "v", "alpha"):
        assert torch.equal(getattr(m, name).grad, getattr(ref, name).grad), name
    # the op's prepared tensors against the device op's
    args = (m.taus, m.direction(), m.alpha, 50.0, 3, True)
    got = torch.ops.ecc_b200.soft_ecc_fwd_host(x.pin_memory(), *args, slab)
    want = torch.ops.ecc_b200.soft_ecc_fwd(x.cuda(), *args)
    for k in (0, 1, 2):   # chi, coefficients, centred field
        assert torch.equal(got[k], want[k]), k


@pytest.mark.parametrize("shape,v,group", [((5, 96, 80), [1.0, 2.0], 2), ((3, 20, 24, 32), [1.0, 2.0, -0.5], 2)])
def test_soft_step_host_streamed_batch_bit_identical(shape, v, group):
    """Batches (2-D, and 3-D with several items) stream in item groups over
    the whole batch's buffers: chi and the gradients equal the device path's
    bit for bit (units sized for a group, one reduction at the end)."""
    B = 256
    u = np.asarray(v) / np.linalg.norm(v)
    span = 0.3 * np.abs(u).sum()
    taus = np.linspace(-span, 1.0 + span, B + 1)[1:]
    x = torch.rand(shape, generator=torch.Generator().manual_seed(5))
    up = torch.rand((shape[0], B), dtype=torch.float64, device="cuda") + 0.5
    ref = E.SoftECC(taus, v, alpha=0.3, lam=50.0).cuda()
    chi_ref = ref(x.cuda())
    (chi_ref * up).sum().backward()
    m = E.SoftECC(taus, v, alpha=0.3, lam=50.0).cuda()
    chi = E.soft_step_host(m, x.pin_memory(), up, micro=group)
    torch.cuda.synchronize()
    assert torch.equal(chi, chi_ref.detach())
    for name in ("taus", "v", "alpha"):
        assert torch.equal(getattr(m, name).grad, getattr(ref, name).grad), name


def test_soft_step_host_without_gradients():
    """Without gradients soft_step_host runs the module over micro-batches
    (the next one's copy overlapping the current one's forward): chi equals
    the device path's, no gradient is touched."""
    x = torch.rand((7, 96, 80), generator=torch.Generator().manual_seed(7))
    m = E.SoftECC(np.linspace(-0.4, 1.4, 64), [1.0, 2.0], alpha=0.3, lam=50.0).cuda()
    with torch.no_grad():
        chi_ref = m(x.cuda())
        chi = E.soft_step_host(m, x.pin_memory(), micro=3)
    torch.cuda.synchronize()
    assert torch.equal(chi, chi_ref)
    assert m.taus.grad is None and m.v.grad is None and m.alpha.grad is None


def test_soft_step_host_3d_item_without_gradients():
    """A single 3-D item without gradients: the streamed forward alone."""
    B, v = 256, [1.0, 2.0, -0.5]
    u = np.asarray(v) / np.linalg.norm(v)
    span = 0.3 * np.abs(u).sum()
    m = E.SoftECC(np.linspace(-span, 1.0 + span, B + 1)[1:], v, alpha=0.3, lam=50.0).cuda()
    x = torch.rand((1, 40, 48, 64), generator=torch.Generator().manual_seed(9))
    with torch.no_grad():
        chi_ref = m(x.cuda())
        chi = E.soft_step_host(m, x.pin_memory(), slab_planes=8)
    torch.cuda.synchronize()
    assert torch.equal(chi, chi_ref)
    assert m.taus.grad is None

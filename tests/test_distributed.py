"""Multi-rank partition logic on CPU (gloo, world sizes 2 and 3).

The slab/halo/all-reduce path of paper_2510_20271_b200.distributed is run
with real torch.distributed collectives over gloo; the per-slab histogram
is the CPU oracle (injected, test-only), so what is checked is the
partition arithmetic, the halo exchange and the reduction: the distributed
histogram must equal the whole-volume histogram bit for bit.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _oracle_hist(view, z0, z1, taus):
    from oracle import oracle

    return torch.from_numpy(oracle.histogram_rows(view.numpy(), z0, z1, taus.taus))


def _worker(rank, world, port, dims, nbins, dtype, result_q):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import oracle
    from paper_2510_20271_b200 import distributed as D
    from paper_2510_20271_b200.grid import ThresholdSet, thresholds_from_range

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        full = oracle.counter_grid(99, dims).reshape(dims)
        if dtype == "u8":
            full = (full * 256).astype(np.uint8)
        z0, z1 = D.slab_bounds(dims[0], world, rank)
        padded = D.alloc_padded_slab(z1 - z0, dims[1:], torch.from_numpy(full[:1]).dtype, "cpu")
        padded[1:-1] = torch.from_numpy(full[z0:z1])
        lo, hi = D.global_range(padded[1:-1].to(torch.float64))
        assert lo == float(full.min()) and hi == float(full.max())
        taus = thresholds_from_range(lo, hi, nbins)
        if dtype == "u8":
            taus = ThresholdSet(np.arange(0.0, 256.0, 7.0))
            hist = D.slab_histogram(padded, taus, hist_fn=lambda v, a, b, t: torch.from_numpy(
                oracle.histogram_rows(v.numpy().astype(np.float64), a, b, t.taus)))
        else:
            hist = D.slab_histogram(padded, taus, hist_fn=_oracle_hist, overlap=True)   # interior sweep overlaps the exchange
            padded[0] = np.nan
            padded[-1] = np.nan
            flat = D.slab_histogram(padded, taus, hist_fn=_oracle_hist)   # exchange, then one sweep (default)
            assert torch.equal(hist, flat)
        curve = D.slab_curve(padded, taus, hist_fn=_oracle_hist if dtype != "u8" else
                             (lambda v, a, b, t: torch.from_numpy(
                                 oracle.histogram_rows(v.numpy().astype(np.float64), a, b, t.taus))))
        if rank == 0:
            bins, ovf = oracle.histogram(full.astype(np.float64) if dtype == "u8" else full, taus.taus)
            ok = np.array_equal(hist.numpy(), np.append(bins, ovf)) and np.array_equal(curve.numpy(), np.cumsum(bins))
            result_q.put(bool(ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,dims,dtype", [(2, (11, 9, 13), "f32"), (3, (10, 17, 6), "f32"),
                                              (2, (7, 5, 40), "u8"), (3, (4, 8, 8), "f32")])
def test_slab_histogram_matches_whole_volume(world, dims, dtype):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, dims, 64, dtype, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    assert q.get(timeout=5) is True


def _soft_item_grads(x, taus, v, alpha, lam, up):
    """(d_tau, d_v, d_alpha) of one item from the oracle (soft.py:199-257 plus
    the alpha gradient), with the module's u = v/|v| reparametrisation."""
    from oracle import oracle

    u = v / np.linalg.norm(v)
    c = oracle.coefficients(oracle.effective_field(x, alpha, u))
    _, dt, _, _, G = oracle.soft_backward(x, c, lam, alpha, u, taus, up)
    du_raw = -alpha * G
    dv = (du_raw - u * (u @ du_raw)) / np.linalg.norm(v)
    return dt, dv, -(G @ u)


def _grad_worker(rank, world, port, result_q):
    """Batch-sharded soft ECC: each rank holds a SoftECC module and its shard of
    the batch, its parameter gradients are the shard's (computed here by the
    CPU oracle, the per-shard kernel being test-injected as for the slabs);
    allreduce_soft_grads must leave every rank with the full batch's."""
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2510_20271_b200 import SoftECC
    from paper_2510_20271_b200 import distributed as D

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(3)
        N, B, lam, alpha = 7, 24, 20.0, 0.3
        xs = rng.random((N, 12, 10))
        v = np.array([1.0, 2.0])
        taus = np.linspace(-0.4, 1.4, B)
        up = rng.uniform(0.5, 1.5, (N, B))
        m = SoftECC(taus, v, alpha=alpha, lam=lam)
        i0, i1 = D.shard_batch(N, world, rank)
        g = [np.zeros(B), np.zeros(2), 0.0]
        for i in range(i0, i1):
            dt, dv, da = _soft_item_grads(xs[i], taus, v, alpha, lam, up[i])
            g = [g[0] + dt, g[1] + dv, g[2] + da]
        m.taus.grad = torch.from_numpy(g[0])
        m.v.grad = torch.from_numpy(g[1])
        m.alpha.grad = torch.tensor(float(g[2]), dtype=torch.float64)
        D.allreduce_soft_grads(m)
        full = [np.zeros(B), np.zeros(2), 0.0]
        for i in range(N):
            dt, dv, da = _soft_item_grads(xs[i], taus, v, alpha, lam, up[i])
            full = [full[0] + dt, full[1] + dv, full[2] + da]
        ok = (np.allclose(m.taus.grad.numpy(), full[0], rtol=1e-12, atol=1e-14)
              and np.allclose(m.v.grad.numpy(), full[1], rtol=1e-12, atol=1e-14)
              and abs(float(m.alpha.grad) - full[2]) <= 1e-12 * max(1.0, abs(full[2])))
        result_q.put((rank, bool(ok), i0, i1))
    finally:
        dist.destroy_process_group()


def test_soft_gradient_allreduce_and_batch_shards():
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_grad_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=5) for _ in range(world))
    assert all(ok for _, ok, _, _ in res)
    spans = [(a, b) for _, _, a, b in res]
    assert spans[0][0] == 0 and spans[-1][1] == 7
    assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))


def _empty_worker(rank, world, port, result_q):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2510_20271_b200 import distributed as D
    from paper_2510_20271_b200.grid import ThresholdSet

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        z0, z1 = D.slab_bounds(2, world, rank)
        padded = D.alloc_padded_slab(z1 - z0, (4, 4), torch.float32, "cpu")
        try:
            D.slab_histogram(padded, ThresholdSet([0.5]), hist_fn=_oracle_hist, depth=2)
            result_q.put((rank, z1 - z0, "ran"))
        except ValueError:
            result_q.put((rank, z1 - z0, "refused"))
    finally:
        dist.destroy_process_group()


def test_more_ranks_than_planes_is_refused():
    """with world > depth an empty rank would hand its neighbours
    uninitialised halo planes; the empty rank refuses before any exchange."""
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_empty_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(60)
    res = sorted(q.get(timeout=5) for _ in range(world))
    assert all(how == "refused" for _, _, how in res) and any(n == 0 for _, n, _ in res)


def test_slab_bounds_cover():
    from paper_2510_20271_b200.distributed import slab_bounds

    for depth in (1, 7, 64, 2048):
        for world in (1, 2, 3, 8):
            spans = [slab_bounds(depth, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == depth
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            assert max(b - a for a, b in spans) - min(b - a for a, b in spans) <= 1


def _file_worker(rank, world, port, path, nbins, result_q):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import oracle
    from paper_2510_20271_b200 import distributed as D
    from paper_2510_20271_b200.grid import thresholds_from_range
    from paper_2510_20271_b200.io import load_slab_device, read_grid

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        # each rank reads its own planes plus the two neighbour planes from the
        # file: no halo exchange (exchange=False)
        padded, (z0, z1) = load_slab_device(path, rank, world, "cpu")
        lo, hi = D.global_range(padded[1:-1].to(torch.float64))
        taus = thresholds_from_range(lo, hi, nbins)
        hist = D.slab_histogram(padded, taus, exchange=False, hist_fn=_oracle_hist)
        if rank == 0:
            full = read_grid(path).values.astype(np.float32)
            bins, ovf = oracle.histogram(full, taus.taus)
            result_q.put(bool(np.array_equal(hist.numpy(), np.append(bins, ovf))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_file_backed_slabs(tmp_path, world):
    """io.load_slab_device + slab_histogram(exchange=False) over gloo equals the
    whole volume's histogram (the file-backed C5 path)."""
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import oracle
    from paper_2510_20271_b200.io import write_grid

    dims = (13, 10, 12)
    path = tmp_path / "v.eccg"
    write_grid(oracle.counter_grid(5, dims).reshape(dims), path)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_file_worker, args=(r, world, port, str(path), 48, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    assert q.get(timeout=5) is True

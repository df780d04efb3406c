"""Multi-GPU partitioning of the ECC hot paths (one process per GPU).

Discrete ECC (BASELINE config C5): the volume is cut into z-slabs (axis 0),
one per rank.  Coefficients need a one-plane halo on each interior side
(the index tie-break is translation invariant, coefficients.py:141-152),
histograms are exactly additive (hard.py:99-118).  So a step is
    halo exchange (send first/last plane to the z-neighbours)
    -> one fused sweep over the own planes (ecc_histogram_range)
    -> all_reduce(SUM) of the (B+1) int64 histogram
    -> prefix scan.
At the two ends of the volume the missing halo plane is simply left out of
the view handed to the kernel, so the grid boundary is the kernel's own.

Soft ECC (C3/C4): batch items are independent, so items are sharded and
only the gradients of the shared parameters (tau, v, alpha) are summed
across ranks (DDP-style all_reduce; ~2 KB).

Everything here goes through torch.distributed, so it runs over NCCL on
GPUs and over gloo on CPU tensors (the multi-process CPU tests inject the
oracle as the per-slab histogram to check the partition logic).
"""

from __future__ import annotations

from typing import Callable

import torch
import torch.distributed as dist


def slab_bounds(depth: int, world: int, rank: int) -> tuple[int, int]:
    """Planes [z0, z1) of rank `rank` for an even split of `depth` planes
    (empty for ranks beyond `depth`; slab_histogram refuses such splits)."""
    base, extra = divmod(depth, world)
    z0 = rank * base + min(rank, extra)
    return z0, z0 + base + (1 if rank < extra else 0)


def alloc_padded_slab(planes: int, plane_shape, dtype, device) -> torch.Tensor:
    """[planes + 2, H, W] buffer: index 0 and -1 are the halo planes."""
    return torch.empty((planes + 2, *plane_shape), dtype=dtype, device=device)


def start_halo_exchange(padded: torch.Tensor, group=None) -> list:
    """Post the sends/receives that fill padded[0] / padded[-1] from the
    z-neighbour ranks; returns the requests (wait on them before reading the
    halo planes).  The own planes padded[1:-1] are only read meanwhile."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    ops = []
    if rank > 0:
        ops.append(dist.P2POp(dist.isend, padded[1].contiguous(), _peer(group, rank - 1), group))
        ops.append(dist.P2POp(dist.irecv, padded[0], _peer(group, rank - 1), group))
    if rank < world - 1:
        ops.append(dist.P2POp(dist.isend, padded[-2].contiguous(), _peer(group, rank + 1), group))
        ops.append(dist.P2POp(dist.irecv, padded[-1], _peer(group, rank + 1), group))
    return dist.batch_isend_irecv(ops) if ops else []


def exchange_halos(padded: torch.Tensor, group=None) -> None:
    """Fill padded[0] / padded[-1] from the z-neighbour ranks.

    padded[1:-1] holds this rank's own planes; the end ranks' outer halo
    planes are left untouched (they are excluded by `slab_view`).
    """
    for req in start_halo_exchange(padded, group):
        req.wait()


def _peer(group, group_rank: int) -> int:
    return group_rank if group is None else dist.get_global_rank(group, group_rank)


def slab_view(padded: torch.Tensor, group=None) -> tuple[torch.Tensor, int, int]:
    """(view, plane_begin, plane_end): the planes the kernel reads and the
    range it deposits.  End ranks drop their (absent) outer halo plane."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    lo = 1 if rank == 0 else 0
    hi = padded.shape[0] - (1 if rank == world - 1 else 0)
    view = padded[lo:hi]
    return view, 1 - lo, 1 - lo + padded.shape[0] - 2


def _cuda_slab_hist(view: torch.Tensor, z0: int, z1: int, taus) -> torch.Tensor:
    from . import _lib

    code = _lib.dtype_code(view)
    table, binning = taus.device_table(code, view.device)
    hist = torch.empty(len(taus) + 1, dtype=torch.int64, device=view.device)
    d = _lib.dims_arg(view.shape)
    _lib.check(_lib.lib().ecc_histogram_range(_lib.ptr(view), code, 3, _lib.ptr(d), 1, z0, z1, _lib.ptr(table),
                                              _lib.ctypes.byref(binning), _lib.ptr(hist), _lib.stream_ptr(view)))
    return hist


def slab_histogram(padded: torch.Tensor, taus, group=None, exchange: bool = True,
                   hist_fn: Callable | None = None, overlap: bool = False, depth: int | None = None) -> torch.Tensor:
    """Global (B+1) int64 histogram of a z-slab-partitioned 3D volume.

    padded: [planes + 2, H, W] (own planes at 1..planes; halos filled here
    when `exchange`).  hist_fn(view, plane_begin, plane_end, taus) -> (B+1)
    int64 histogram of planes [plane_begin, plane_end) of the contiguous
    view; defaults to the CUDA kernel (ecc_histogram_range).

    depth (the volume's plane count, optional): every rank refuses a split
    with more ranks than planes before any collective, so all of them raise
    together; without it only the empty rank raises (an empty
    rank's halo slots would otherwise reach its neighbours as their boundary
    planes).

    overlap (with exchange, >= 3 own planes, >1 rank): the interior planes
    [1, planes - 1) need only this rank's own data, so they are swept while
    the halo planes are in flight; the two boundary planes follow once the
    halos have arrived.  Histograms are additive over plane ranges, so the
    sum equals the single sweep bit for bit.  Off by default: a one-plane
    sweep is a whole launch (setup, counter zeroing and flush of every
    CTA), 31.6 us at 512^2 planes against 240 us for the 512-plane slab
    (tools/plane_sweep.py), while the two halo planes cross NVLink in a few
    microseconds -- exchanging first and sweeping once is cheaper.
    """
    fn = hist_fn or _cuda_slab_hist
    planes = padded.shape[0] - 2
    if (depth is not None and depth < dist.get_world_size(group)) or planes < 1:
        raise ValueError("every rank needs at least one plane (more ranks than planes in the volume)")
    if exchange and overlap and planes >= 3 and dist.get_world_size(group) > 1:
        reqs = start_halo_exchange(padded, group)
        hist = fn(padded[1:-1], 1, planes - 1, taus)
        for req in reqs:
            req.wait()
        view, z0, z1 = slab_view(padded, group)
        hist = hist + fn(view, z0, z0 + 1, taus) + fn(view, z1 - 1, z1, taus)
    else:
        if exchange:
            exchange_halos(padded, group)
        view, z0, z1 = slab_view(padded, group)
        hist = fn(view, z0, z1, taus)
    dist.all_reduce(hist, op=dist.ReduceOp.SUM, group=group)
    return hist


def slab_curve(padded: torch.Tensor, taus, group=None, hist_fn: Callable | None = None,
               depth: int | None = None) -> torch.Tensor:
    """Exact int64 ECC curve [B] of the whole distributed volume (every rank)."""
    hist = slab_histogram(padded, taus, group, hist_fn=hist_fn, depth=depth)
    return torch.cumsum(hist[:-1], 0) if not hist.is_cuda else _scan(hist, len(taus))


def _scan(hist: torch.Tensor, nb: int) -> torch.Tensor:
    from .hard import scan_device

    return scan_device(hist.reshape(1, -1), nb)[0]


def global_range(x: torch.Tensor, group=None) -> tuple[float, float]:
    """(min, max) over all ranks' own data (uniform_thresholds, grid.py:192-193)."""
    if x.is_cuda:
        from .hard import device_minmax

        lo, hi, _ = device_minmax(x)
    else:
        lo, hi = float(x.min()), float(x.max())
    t = torch.tensor([-lo, hi], dtype=torch.float64, device=x.device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return -float(t[0]), float(t[1])


def shard_batch(n_items: int, world: int, rank: int) -> tuple[int, int]:
    """Items [i0, i1) of this rank for batch-sharded soft ECC."""
    return slab_bounds(n_items, world, rank)


def allreduce_soft_grads(module: torch.nn.Module, group=None) -> None:
    """Sum the shared-parameter gradients (tau, v, alpha) across ranks."""
    grads = [p.grad for p in module.parameters() if p.grad is not None]
    if not grads:
        return
    flat = torch.cat([g.reshape(-1).to(torch.float64) for g in grads])
    dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)
    off = 0
    for g in grads:
        n = g.numel()
        g.copy_(flat[off:off + n].reshape(g.shape).to(g.dtype))
        off += n

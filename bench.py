"""Benchmark of the B200 ECC engine (driver contract: one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Headline workload (BASELINE.json configs[1], the metric's 1-GPU config):
discrete ECC of a 3D 512^3 float32 volume with 1024 uniform thresholds.
Under torchrun with N ranks the volume is z-slab sharded (weak scaling: each
rank owns 512 planes of 512x512, a one-plane halo is exchanged with the
z-neighbours over NCCL and the (B+1) int64 histogram is all-reduced), i.e.
the C5 pipeline at 512 planes per GPU.

A step = one pass of the hot path over the volume: halo exchange (N>1) +
fused stencil/bin/histogram sweep + all-reduce (N>1) + prefix scan.  Inputs
are resident in HBM and larger than L2 (512 MiB per rank vs 126 MB), so no
flush is needed between steps.  `e2e` repeats the measurement through the
public API with the volume copied host->device from pinned memory every step
and the curve copied back.  `soft` reports the C3 soft-ECC forward+backward
(128 x 1024^2, 256 thresholds, lambda 50, learnable tau/u/alpha).

--impl reference times the reference algorithm's CPU port (oracle/, all host
threads) on a bounded sample of the same workload (the reference is pure
Python/numpy and cannot travel to the GPU box; its C restatement is pinned
to the reference's golden vectors, see tests/test_oracle_golden.py).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "ECC Gvoxels/s (discrete, 3D f32, 1024 bins)"
UNIT = "Gvoxel/s"
NB = 1024
SEED = 20261018


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={','.join(self.FIELDS)}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(self.index)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.3)
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.2)
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) != 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def _dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ---------------------------------------------------------------------------
# reference arm: the CPU port on a bounded sample
# ---------------------------------------------------------------------------

def cpu_port_sample(planes: int = 32, reps: int = 1):
    """Time oracle/ (the C restatement of ecckit's compute_ecc, all host
    threads) on `planes` planes of the 512^3 workload.  Returns Gvox/s."""
    from oracle import oracle

    dims = (planes + 2, 512, 512)
    x = oracle.counter_grid(SEED, dims).reshape(dims)
    taus = np.linspace(0.0, 1.0, NB + 1)[1:]
    oracle.histogram_rows(x, 1, planes + 1, taus)  # warm-up (thread pool)
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        oracle.histogram_rows(x, 1, planes + 1, taus)
        ts.append(time.perf_counter() - t0)
    vox = planes * 512 * 512
    return vox / min(ts) / 1e9, oracle.num_threads(), f"{planes}x512x512 f32 planes of the 512^3 volume, {NB} bins"


def run_reference(args):
    world, rank, _ = _dist_env()
    if rank != 0:
        return
    vals = []
    sample = ""
    cores = 1
    for _ in range(args.warmup):
        cpu_port_sample(planes=16)
    for _ in range(args.steps):
        v, cores, sample = cpu_port_sample(planes=32)
        vals.append(v)
    value = statistics.median(vals)
    vox_per_step = 512 * 512 * 512 * world
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": vox_per_step / (value * 1e9) * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": "C2: 3D 512^3 float32 volume, discrete ECC, 1024 uniform thresholds "
                   "(sampled: 32 planes per step)", "volume": [512 * world, 512, 512], "bins": NB,
                   "parallelism": f"zslab{world}"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------

def run_b200(args):
    import torch
    import torch.distributed as dist

    import paper_2510_20271_b200 as E
    from paper_2510_20271_b200 import _lib
    from paper_2510_20271_b200 import distributed as D

    world, rank, local = _dist_env()
    # ECC_BENCH_FORCE_DIST=1 runs the multi-GPU code path (NCCL, halo exchange,
    # all-reduces) even with one rank: a one-GPU check of the N > 1 plumbing
    dist_on = world > 1 or os.environ.get("ECC_BENCH_FORCE_DIST") == "1"
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if dist_on:
        dist.init_process_group("nccl", device_id=dev)
    L = _lib.lib()
    stream = torch.cuda.current_stream(dev)

    # --- synthetic volume: this rank's 512 planes (+ halos) --------------------
    P, H, W = args.planes, 512, 512
    padded = D.alloc_padded_slab(P, (H, W), torch.float32, dev)
    own = padded[1:-1]
    start = rank * P * H * W
    _lib.check(L.ecc_counter_grid(SEED, start, own.numel(), _lib.ptr(own), _lib.stream_ptr(own)))

    # thresholds: uniform over the global range (device min/max, grid.py:183-196)
    torch.cuda.synchronize()
    for _ in range(2):  # second call timed (first pays lazy init)
        t0 = time.perf_counter()
        if dist_on:
            lo, hi = D.global_range(own)
        else:
            lo, hi, _ = E.device_minmax(own)
        torch.cuda.synchronize()
        minmax_ms = (time.perf_counter() - t0) * 1e3
    # device time of the min/max pass alone (K4; CUDA events, no host sync inside)
    mm_out = torch.empty(3, dtype=torch.int64, device=dev)
    m0, m1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    m0.record(stream)
    for _ in range(5):
        _lib.check(L.ecc_minmax(_lib.ptr(own), _lib.DTYPE_F32, own.numel(), _lib.ptr(mm_out),
                                _lib.ctypes.c_void_p(stream.cuda_stream)))
    m1.record(stream)
    torch.cuda.synchronize()
    minmax_kernel_ms = m0.elapsed_time(m1) / 5
    taus = E.thresholds_from_range(lo, hi, NB)
    table, binning = taus.device_table(_lib.DTYPE_F32, dev)
    hist = torch.empty(NB + 1, dtype=torch.int64, device=dev)
    curve = torch.empty(NB, dtype=torch.int64, device=dev)
    view, z0, z1 = (own, 0, P) if not dist_on else D.slab_view(padded)
    dims = _lib.dims_arg(view.shape)
    # kernel-only timing: one event pair per step around the histogram kernel,
    # steps back to back (no host sync in between), read after the last one
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    kernel_ms = []

    dims_cache = {tuple(view.shape): dims}

    def sweep(v, a, b, out):
        dv = dims_cache.get(tuple(v.shape))
        if dv is None:
            dv = dims_cache[tuple(v.shape)] = _lib.dims_arg(v.shape)
        _lib.check(L.ecc_histogram_range(_lib.ptr(v), _lib.DTYPE_F32, 3, _lib.ptr(dv), 1, a, b,
                                         _lib.ptr(table), _lib.ctypes.byref(binning), _lib.ptr(out),
                                         _lib.ctypes.c_void_p(stream.cuda_stream)))
        return out

    def slab_fn(v, a, b, t):
        return sweep(v, a, b, torch.empty(NB + 1, dtype=torch.int64, device=dev))

    def step(record=None):
        if record is not None:
            # kernel-only pass: the fused sweep over this rank's planes, no collectives
            kstart, kend = kev[record]
            kstart.record(stream)
            sweep(view, z0, z1, hist)
            kend.record(stream)
            return
        if dist_on:
            # halo exchange in flight while the interior planes are swept, then
            # the two boundary planes, histogram all-reduce (distributed.slab_histogram)
            h = D.slab_histogram(padded, taus, hist_fn=slab_fn)
        else:
            h = sweep(view, z0, z1, hist)
        _lib.check(L.ecc_scan(_lib.ptr(h), 1, NB, _lib.ptr(curve), _lib.ctypes.c_void_p(stream.cuda_stream)))
        return h

    # correctness gate on the real workload (size-independent properties):
    # the full-volume curve ends at chi(box) = 1 and sums of c are 1.
    h = step().cpu().numpy()
    c = curve.cpu().numpy()
    assert int(h.sum()) == 1 and int(c[-1]) == 1, "ECC invariant violated (sum c != 1)"
    checksum = int(np.bitwise_xor.reduce(c.view(np.uint64)))

    def barrier():
        if dist_on:
            dist.barrier(device_ids=[local])
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    barrier()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        barrier()
    total_ms = ev0.elapsed_time(ev1)
    # kernel-only timing of the dominant kernel (same stream, separate pass)
    for i in range(args.steps):
        step(record=i)
    torch.cuda.synchronize()
    kernel_ms = [a.elapsed_time(b) for a, b in kev]
    if dist_on:
        t = torch.tensor([total_ms, statistics.mean(kernel_ms)], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms, kmean = float(t[0]), float(t[1])
    else:
        kmean = statistics.mean(kernel_ms)
    ms_per_step = total_ms / args.steps
    vox_rank = P * H * W
    vox_total = vox_rank * world
    value = vox_total / (ms_per_step * 1e-3) / 1e9

    peak, peak_kind = _peaks()
    achieved = 4.0 * vox_rank / (kmean * 1e-3) / 1e9
    traffic = None
    tfile = ROOT / "profiles" / "ncu_traffic.json"
    if tfile.exists():
        try:
            traffic = json.loads(tfile.read_text()).get("bytes_per_launch")
        except (ValueError, OSError):
            traffic = None

    # --- e2e through the public API: pinned H2D + compute + D2H -------------
    e2e = None
    if not args.no_e2e:
        # every step: this rank's slab pinned host -> HBM, the public API call,
        # curve HBM -> host (N = 1: ecc_discrete_host; N > 1: distributed.slab_curve,
        # which adds the halo exchange and the histogram all-reduce)
        host = torch.empty((P, H, W), dtype=torch.float32, pin_memory=True)
        host.copy_(own.cpu())
        if not dist_on:
            def e2e_step():
                return E.ecc_discrete_host(host, taus, chunk_planes=64).cpu()
            api = ("paper_2510_20271_b200.ecc_discrete_host (resident layout, 64-plane chunks: every plane "
                   "crosses PCIe once; the planes already on the device are deposited while the next chunk "
                   "is copied)")
        else:
            buf = D.alloc_padded_slab(P, (H, W), torch.float32, dev)

            def e2e_step():
                buf[1:-1].copy_(host, non_blocking=True)
                return D.slab_curve(buf, taus).cpu()
            api = "paper_2510_20271_b200.distributed.slab_curve"

        got = e2e_step()
        assert int(got[-1]) == 1
        for _ in range(2):
            e2e_step()
        barrier()
        reps = max(3, min(args.steps, 10))
        t0 = time.perf_counter()
        for _ in range(reps):
            e2e_step()
        barrier()
        e_ms = (time.perf_counter() - t0) * 1e3 / reps
        if dist_on:
            t = torch.tensor([e_ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms = float(t[0])
        e2e = {"value": vox_total / (e_ms * 1e-3) / 1e9, "unit": UNIT, "ms_per_step": e_ms,
               "h2d_bytes_per_step": int(host.numel() * 4) * world, "d2h_bytes_per_step": int(NB * 8) * world,
               "api": api + " (pinned host -> HBM copy inside the timed region)"}
        del host

    # --- north-star volume (1024^3 f32, 1024 bins; N = 1 only) ---------------
    ns = None
    if world == 1 and not args.no_ns:
        ns = bench_ns(args, dev)

    # --- soft ECC C3 (forward + backward) -------------------------------------
    soft = None
    if not args.no_soft:
        soft = bench_soft(args, dev, world, rank, dist_on)

    # --- C5 per-GPU slab and C4 (one 1024^3 soft item per GPU) -----------------
    c5 = None if args.no_c5 else bench_c5_slab(args, dev, world, rank, dist_on)
    c4 = None if args.no_soft or args.no_c4 else bench_c4(args, dev, world, rank, dist_on)

    # --- CPU baseline (rank 0, N = 1) ----------------------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        v, cores, sample = cpu_port_sample(planes=32)
        cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": "C2: 3D 512^3 float32 volume, discrete ECC, 1024 uniform thresholds"
                       + (" (z-slab per GPU, halo exchange + NCCL histogram all-reduce)" if dist_on else ""),
                       "volume": [P * world, H, W], "bins": NB, "parallelism": f"zslab{world}",
                       "l2": "input larger than L2 (512 MiB per GPU), no flush",
                       "thresholds": "given (uniform over the device min/max, computed once)",
                       "minmax_pass_ms": minmax_ms, "minmax_kernel_ms": minmax_kernel_ms,
                       "minmax_kernel_gbs": 4.0 * own.numel() / (minmax_kernel_ms * 1e-3) / 1e9, "seed": SEED, "curve_xor_checksum": checksum},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_kind,
                         "kernel": "ecc_fast3d_bin_kernel" if W % 4 == 0 else "ecc_sweep_kernel<RawSrc<float>,HistSink<float>>",
                         "kernel_ms": kmean, "algorithmic_bytes_per_launch": 4 * vox_rank},
            "cpu_baseline": cpu,
            "e2e": e2e,
            # per step: the sweep (three with the overlapped halo exchange at N > 1) + the scan
            "gpu_launches": (4 if world > 1 and P >= 3 else 2) * args.steps,
            "clocks": clocks.summary(),
            "north_star": ns,
            "soft": soft,
            "c4": c4,
            "c5_slab": c5,
        }
        print(json.dumps(line), flush=True)
    if dist_on:
        dist.destroy_process_group()


def bench_ns(args, dev):
    """The north-star case on one GPU: 1024^3 float32, 1024 uniform thresholds,
    device-resident input (4 GiB > L2), CUDA-event timing over K steps.  The
    curve is checked against the size-independent invariants (sum c = 1)."""
    import torch

    import paper_2510_20271_b200 as E
    from paper_2510_20271_b200 import _lib

    L = _lib.lib()
    n = 1024
    x = torch.empty((n, n, n), dtype=torch.float32, device=dev)
    _lib.check(L.ecc_counter_grid(SEED + 1, 0, x.numel(), _lib.ptr(x), _lib.stream_ptr(x)))
    lo, hi, _ = E.device_minmax(x)
    taus = E.thresholds_from_range(lo, hi, NB)
    curve, hist = E.ecc_discrete(x, taus, return_hist=True)
    assert int(hist.sum()) == 1 and int(curve[-1]) == 1, "ECC invariant violated at 1024^3"
    for _ in range(3):
        E.histogram_device(x, taus)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    steps = max(3, min(args.steps, 10))
    e0.record()
    for _ in range(steps):
        E.histogram_device(x, taus)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    peak, peak_kind = _peaks()
    gbs = 4.0 * x.numel() / (ms * 1e-3) / 1e9
    traffic = None
    tfile = ROOT / "profiles" / "ncu_traffic.json"
    if tfile.exists():
        try:
            t = json.loads(tfile.read_text()).get("north_star", {})
            traffic = t["dram_read_bytes"] + t["dram_write_bytes"]
        except (ValueError, OSError, KeyError):
            traffic = None
    out = {"workload": "NS: 3D 1024^3 float32, discrete ECC, 1024 uniform thresholds (device-resident)",
           "value": x.numel() / (ms * 1e-3) / 1e9, "unit": UNIT, "ms_per_step": ms, "steps": steps,
           "roofline": {"bound": "hbm", "achieved": gbs, "peak": peak, "unit": "GB/s", "frac": gbs / peak,
                        "peak_source": peak_kind, "traffic": traffic,
                        "algorithmic_bytes_per_launch": 4 * x.numel()}}
    del x
    torch.cuda.empty_cache()
    return out


def bench_c5_slab(args, dev, world, rank, dist_on=False):
    """One GPU's share of C5 (3D 2048^3 float32, z-slabs over 8 GPUs): a
    256 x 2048 x 2048 slab (4 GiB) of the counter-generated C5 volume (the
    planes rank r would own in an 8-way split, r = this rank mod 8) plus its
    two halo planes, swept by the fused kernel over its own planes
    (ecc_histogram_range, the per-rank kernel of distributed.slab_histogram).
    Thresholds: 1024 uniform over [0, 1) edges of the generator's range.
    The halo exchange and the 8 KiB histogram all-reduce are timed by the
    multi-GPU C2 line; here the slab kernel alone, CUDA events."""
    import torch

    import paper_2510_20271_b200 as E
    from paper_2510_20271_b200 import _lib
    from paper_2510_20271_b200 import distributed as D

    L = _lib.lib()
    P, H, W = 256, 2048, 2048
    part = rank % 8
    padded = D.alloc_padded_slab(P, (H, W), torch.float32, dev)
    z0 = part * P
    lo_plane = max(z0 - 1, 0)
    hi_plane = min(z0 + P + 1, 8 * P)
    first = 1 - (z0 - lo_plane)
    view = padded[first:first + (hi_plane - lo_plane)]
    _lib.check(L.ecc_counter_grid(SEED + 2, lo_plane * H * W, view.numel(), _lib.ptr(view), _lib.stream_ptr(view)))
    taus = E.thresholds_from_range(0.0, 1.0 - 2.0 ** -24, NB)
    table, binning = taus.device_table(_lib.DTYPE_F32, dev)
    hist = torch.zeros(NB + 1, dtype=torch.int64, device=dev)
    zlo, zhi = z0 - lo_plane, z0 - lo_plane + P
    dims = _lib.dims_arg(view.shape)
    stream = torch.cuda.current_stream(dev)

    def run():
        _lib.check(L.ecc_histogram_range(_lib.ptr(view), _lib.DTYPE_F32, 3, _lib.ptr(dims), 1, zlo, zhi,
                                         _lib.ptr(table), _lib.ctypes.byref(binning), _lib.ptr(hist),
                                         _lib.ctypes.c_void_p(stream.cuda_stream)))

    run()
    torch.cuda.synchronize()
    for _ in range(2):
        run()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    steps = max(3, min(args.steps, 10))
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(steps):
        run()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    if dist_on:
        import torch.distributed as dist

        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t[0])
    peak, peak_kind = _peaks()
    vox = P * H * W
    gbs = 4.0 * vox / (ms * 1e-3) / 1e9
    out = {"workload": "C5 per-GPU slab: planes [%d, %d) of the 2048^3 float32 counter volume (+ halos), "
                       "1024 thresholds, fused slab kernel (ecc_histogram_range)" % (z0, z0 + P),
           "value": vox * world / (ms * 1e-3) / 1e9, "unit": UNIT, "ms_per_step": ms, "steps": steps,
           "n_gpus": world, "scaling": "weak",
           "roofline": {"bound": "hbm", "achieved": gbs, "peak": peak, "unit": "GB/s", "frac": gbs / peak,
                        "peak_source": peak_kind}}
    del padded, view
    torch.cuda.empty_cache()
    return out


def bench_c4(args, dev, world, rank, dist_on=False):
    """C4: 3D 1024^3 float32 soft ECC, forward + backward, learnable tau / v /
    alpha, batch-sharded (one item per GPU), B = 256, lambda = 50, alpha =
    0.3, u = normalize(1, 2, -0.5); the shared parameters'
    gradients are all-reduced under torchrun (distributed.allreduce_soft_grads)."""
    import torch

    import paper_2510_20271_b200 as E

    n, B, lam, alpha = 1024, 256, 50.0, 0.3
    g = torch.Generator(device=dev)
    g.manual_seed(SEED + 100 + rank)
    x = torch.rand((1, n, n, n), device=dev, generator=g, dtype=torch.float32)
    v = np.array([1.0, 2.0, -0.5])
    u = v / np.linalg.norm(v)
    span = alpha * np.abs(u).sum()
    m = E.SoftECC(np.linspace(-span, 1.0 + span, B + 1)[1:], v, alpha=alpha, lam=lam).to(dev)
    up = torch.ones((1, B), dtype=torch.float64, device=dev)

    def step():
        m.zero_grad(set_to_none=True)
        m(x).backward(up)
        if dist_on:
            from paper_2510_20271_b200 import distributed as D

            D.allreduce_soft_grads(m)

    step()
    torch.cuda.synchronize()
    steps = 2
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    if dist_on:
        import torch.distributed as dist

        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t[0])
    assert bool(torch.isfinite(m.taus.grad).all()), "non-finite d_tau at C4"
    vox = n ** 3 * world
    out = {"workload": "C4: 3D 1024^3 float32 soft ECC fwd+bwd, learnable tau/u/alpha, one item per GPU",
           "value": vox / (ms * 1e-3), "unit": "voxel/s", "ms_per_step": ms, "steps": steps,
           "n_gpus": world, "bins": B, "lambda": lam, "alpha": alpha, "parallelism": f"batch{world}",
           "algorithmic_pairs_per_s": 2 * vox * B / (ms * 1e-3)}
    del x, m
    torch.cuda.empty_cache()
    return out


def bench_soft(args, dev, world, rank, dist_on=False):
    import torch

    import paper_2510_20271_b200 as E

    N, H, W, B, lam, alpha = args.soft_batch, 1024, 1024, 256, 50.0, 0.3
    g = torch.Generator(device=dev)
    g.manual_seed(SEED + rank)
    x = torch.rand((N, H, W), device=dev, generator=g, dtype=torch.float32)
    v = np.array([1.0, 2.0])
    u = v / np.linalg.norm(v)
    span = alpha * np.abs(u).sum()
    taus = np.linspace(-span, 1.0 + span, B + 1)[1:]
    m = E.SoftECC(taus, v, alpha=alpha, lam=lam).to(dev)
    up = torch.ones((N, B), dtype=torch.float64, device=dev)

    def step():
        m.zero_grad(set_to_none=True)
        chi = m(x)
        chi.backward(up)
        if dist_on:
            from paper_2510_20271_b200 import distributed as D

            D.allreduce_soft_grads(m)

    step()
    torch.cuda.synchronize()
    steps = max(2, min(args.steps, 5))
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    if dist_on:
        import torch.distributed as dist

        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t[0])
    # fraction of voxels with c != 0 (the kernels skip the others)
    from paper_2510_20271_b200 import soft as S

    p = S._params(lam, alpha, u, float(taus[0]), float(taus[-1]), 2, S._block_halfwidth(taus))
    c0, _ = S.soft_prepare_device(x[:8].contiguous(), (H, W), min(N, 8), p)
    nz = float(torch.count_nonzero(c0)) / c0.numel()
    vox = N * H * W * world
    pairs = vox * B * 2                      # algorithmic (voxel, threshold) pairs, forward + backward
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    mufu_peak = 16 * sms * 1.965e9 * world   # MUFU.RCP lane-ops/s (15.9/clk/SM measured, tools/microbench)
    # MUFU work actually issued: the kernels evaluate only c != 0 voxels; the
    # forward takes one reciprocal per two pairs (paired denominators), the
    # backward 7/8 per pair (1/8 as Newton steps on the FMA pipe); plus one
    # ex2 per voxel and lane (T = 16)
    mufu_ops = nz * vox * B * ((0.5 + 1.0 / 16.0) + (7.0 / 8.0 + 1.0 / 16.0))
    return {"metric": "soft-ECC fwd+bwd voxels/s", "value": vox / (ms * 1e-3), "unit": "voxel/s",
            "ms_per_step": ms, "steps": steps,
            "config": {"workload": "C3: batched 2D 128x1024x1024 f32, soft ECC fwd+bwd, learnable tau/u/alpha",
                       "batch_per_gpu": N, "bins": B, "lambda": lam, "alpha": alpha, "parallelism": f"batch{world}"},
            "roofline": {"bound": "sfu", "unit": "MUFU ops/s", "achieved": mufu_ops / (ms * 1e-3),
                         "peak": mufu_peak, "frac": mufu_ops / (ms * 1e-3) / mufu_peak,
                         "nonzero_fraction": nz, "algorithmic_pairs_per_s": pairs / (ms * 1e-3),
                         # one MUFU per (voxel, threshold) pair per pass bounds fwd+bwd at
                         # mufu_peak / (2 B) voxels/s; skipping c = 0 voxels and pairing reciprocals beat it
                         "survey_sfu_bound_voxel_s": mufu_peak / (2 * B),
                         "vs_survey_sfu_bound": (vox / (ms * 1e-3)) / (mufu_peak / (2 * B)),
                         "mufu_per_executed_pair": {"forward": 0.5, "backward": 7.0 / 8.0},
                         "note": "achieved counts the MUFU operations the kernels issue (c = 0 voxels are "
                                 "skipped; the forward pairs its reciprocals, one per two pairs; 1/8 of the "
                                 "backward's run as Newton steps on the FMA pipe)"}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--planes", type=int, default=512, help="planes per GPU (512 = C2)")
    ap.add_argument("--soft-batch", type=int, default=128)
    ap.add_argument("--no-soft", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-ns", action="store_true", help="skip the 1024^3 north-star measurement")
    ap.add_argument("--no-c4", action="store_true", help="skip the 1024^3 soft (C4) measurement")
    ap.add_argument("--no-c5", action="store_true", help="skip the C5 per-GPU slab measurement")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()

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
and the curve copied back.

Further legs (sub-objects of the line): `north_star` (1024^3 on one GPU),
`c5` (the 2048^3 volume z-slab sharded over the N ranks, strong scaling),
`soft` (C3: 128 x 1024^2, 256 thresholds, lambda 50, learnable tau/u/alpha,
forward + backward, batch-sharded) and `c4` (one 1024^3 soft item per GPU).
Every leg is gated on the CPU oracle before its time is reported
(`parity`), as the reference's own harness refuses to time a wrong answer
(/root/reference/pkg/src/ecckit/bench.py:28-37, 115-117).

--impl reference times the reference algorithm's CPU port (oracle/, all host
threads) on the full C2 volume every step (the reference is pure
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
# reference arm and CPU baselines: the CPU port (oracle/, the checker) timed
# on the box's host cores on the same full volume
# ---------------------------------------------------------------------------

def cpu_port_c2(planes: int = 512, threads: int | None = None, reps: int = 1):
    """Time oracle/ (the C restatement of ecckit's compute_ecc) on the full
    C2 volume (`planes` x 512 x 512 float32 counter grid, SEED, 1024 uniform
    thresholds over [0, 1)) with `threads` OpenMP threads (None: all host
    threads; the reference's `workers`, hard.py:184-200).  Returns
    (Gvox/s of the best rep, threads, sample text, bins+overflow)."""
    from oracle import oracle

    nthreads = threads or os.cpu_count() or 1
    oracle.set_threads(nthreads)
    dims = (planes, 512, 512)
    x = oracle.counter_grid(SEED, dims).reshape(dims)
    taus = np.linspace(0.0, 1.0, NB + 1)[1:]
    ts = []
    hist = None
    for _ in range(reps):
        t0 = time.perf_counter()
        bins, ovf = oracle.histogram(x, taus)
        ts.append(time.perf_counter() - t0)
        hist = np.concatenate([bins, [ovf]])
    oracle.set_threads(os.cpu_count() or 1)
    vox = planes * 512 * 512
    return (vox / min(ts) / 1e9, nthreads,
            f"full {planes}x512x512 f32 volume, {NB} bins, {nthreads} OpenMP threads", hist)


def run_reference(args):
    world, rank, _ = _dist_env()
    if rank != 0:
        return
    planes = 512 * world
    for _ in range(args.warmup):
        cpu_port_c2(planes)
    vals = []
    cores, sample = 1, ""
    for _ in range(args.steps):
        v, cores, sample, _ = cpu_port_c2(planes)
        vals.append(v)
    value = statistics.median(vals)
    vox_per_step = 512 * 512 * planes
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": vox_per_step / (value * 1e9) * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": "C2: 3D 512^3 float32 volume, discrete ECC, 1024 uniform thresholds "
                   "(full volume every step)", "volume": [planes, 512, 512], "bins": NB,
                   "parallelism": f"zslab{world}"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_soft_sample(ndim: int, reps: int = 1):
    """The oracle's soft forward + backward (soft.py:154-257, float64, all host
    threads) on one C3 image (1024 x 1024, ndim = 2) or a 128^3 C4 sub-volume
    (ndim = 3), B = 256, lambda = 50, alpha = 0.3.  Returns (voxels/s, threads,
    sample text, voxels of the sample)."""
    from oracle import oracle

    rng = np.random.default_rng(SEED)
    B, lam, alpha = 256, 50.0, 0.3
    v = np.array([1.0, 2.0]) if ndim == 2 else np.array([1.0, 2.0, -0.5])
    u = v / np.linalg.norm(v)
    span = alpha * np.abs(u).sum()
    taus = np.linspace(-span, 1.0 + span, B + 1)[1:]
    dims = (1024, 1024) if ndim == 2 else (128, 128, 128)
    x = rng.random(dims).astype(np.float32).astype(np.float64)
    up = np.ones(B)
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        c = oracle.coefficients(oracle.effective_field(x, alpha, u))
        oracle.soft_forward(x, c, lam, alpha, u, taus)
        oracle.soft_backward(x, c, lam, alpha, u, taus, up)
        ts.append(time.perf_counter() - t0)
    n = int(np.prod(dims))
    what = "one 1024x1024 C3 image" if ndim == 2 else "a 128^3 sub-volume of the C4 item"
    return (n / min(ts), oracle.num_threads(),
            f"{what}, B = 256, forward + backward in float64; voxels/s extrapolated linearly in voxels "
            "(the work per (voxel, threshold) pair is uniform)", n)


# ---------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------

def _gate(ok: bool, what: str):
    """The reference harness never reports a time for a wrong answer
    (/root/reference/pkg/src/ecckit/bench.py:28-37, 115-117)."""
    if not ok:
        raise SystemExit(f"bench: parity gate failed ({what}); no number is reported")


def _max_over_ranks(vals, dev, dist_on):
    if not dist_on:
        return vals
    import torch
    import torch.distributed as dist

    t = torch.tensor(vals, dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(v) for v in t]


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
    if dist_on:   # halo planes of the global volume (timed steps exchange them again)
        D.exchange_halos(padded)

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
    # kernel-only timing: one event pair per step around the histogram kernel,
    # steps back to back (no host sync in between), read after the last one
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    dims_cache = {}

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
            # halo exchange, one sweep over the own planes, histogram all-reduce
            # (distributed.slab_histogram)
            h = D.slab_histogram(padded, taus, hist_fn=slab_fn, depth=P * world)
        else:
            h = sweep(view, z0, z1, hist)
        _lib.check(L.ecc_scan(_lib.ptr(h), 1, NB, _lib.ptr(curve), _lib.ctypes.c_void_p(stream.cuda_stream)))
        return h

    # parity gate on the timed workload: the global histogram of the (world x
    # 512)-plane volume equals the oracle's, bit for bit (rank 0 checks)
    h = step().cpu().numpy()
    c = curve.cpu().numpy()
    _gate(int(h.sum()) == 1 and int(c[-1]) == 1, "C2 sum of coefficients")
    parity = "invariants only"
    if rank == 0 and not args.no_parity:
        from oracle import parity as OP

        want = OP.counter_slab_hist(SEED, (P * world, H, W), 0, P * world, taus.taus)
        _gate(np.array_equal(h, want), "C2 histogram vs oracle")
        parity = "checked: bit-exact vs the CPU oracle on the timed volume"
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
    total_ms, kmean = _max_over_ranks([total_ms, statistics.mean(kernel_ms)], dev, dist_on)
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
        _gate(int(got[-1]) == 1 and np.array_equal(got.numpy(), c), "C2 e2e curve")
        for _ in range(2):
            e2e_step()
        barrier()
        reps = max(3, min(args.steps, 10))
        t0 = time.perf_counter()
        for _ in range(reps):
            e2e_step()
        barrier()
        e_ms = (time.perf_counter() - t0) * 1e3 / reps
        e_ms = _max_over_ranks([e_ms], dev, dist_on)[0]
        e2e = {"value": vox_total / (e_ms * 1e-3) / 1e9, "unit": UNIT, "ms_per_step": e_ms,
               "h2d_bytes_per_step": int(host.numel() * 4) * world, "d2h_bytes_per_step": int(NB * 8) * world,
               "api": api + " (pinned host -> HBM copy inside the timed region)"}
        del host
    del padded, own, view
    torch.cuda.empty_cache()

    # --- north-star volume (1024^3 f32, 1024 bins; N = 1 only) ---------------
    ns = None
    if world == 1 and not args.no_ns:
        ns = bench_ns(args, dev)

    # --- C5: 2048^3 z-slabs over the N ranks (strong scaling) ------------------
    c5 = None if args.no_c5 else bench_c5(args, dev, world, rank, dist_on)

    # --- soft ECC C3 (forward + backward) and C4 (one 1024^3 item per GPU) ------
    soft = None if args.no_soft else bench_soft(args, dev, world, rank, dist_on)
    c4 = None if args.no_soft or args.no_c4 else bench_c4(args, dev, world, rank, dist_on)

    # --- CPU baseline (rank 0, N = 1): the oracle port on the full C2 volume ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        v, cores, sample, cpu_hist = cpu_port_c2(P)
        v1, _, sample1, _ = cpu_port_c2(P, threads=1)
        cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample,
               "workers_1": {"value": v1, "unit": UNIT, "cores": 1, "sample": sample1},
               "same_config": True}

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
                       "minmax_kernel_gbs": 4.0 * vox_rank / (minmax_kernel_ms * 1e-3) / 1e9, "seed": SEED,
                       "curve_xor_checksum": checksum},
            "parity": parity,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_kind,
                         "kernel": "ecc_rank4_kernel" if W % 128 == 0 else "ecc_fast3d_bin_kernel",
                         "kernel_ms": kmean, "algorithmic_bytes_per_launch": 4 * vox_rank},
            "cpu_baseline": cpu,
            "e2e": e2e,
            # per step: the slab sweep + the scan (the halo exchange and the all-reduce are NCCL's)
            "gpu_launches": 2 * args.steps,
            "clocks": clocks.summary(),
            "north_star": ns,
            "c5": c5,
            "soft": soft,
            "c4": c4,
        }
        print(json.dumps(line), flush=True)
    if dist_on:
        dist.destroy_process_group()


def bench_ns(args, dev):
    """The north-star case on one GPU: 1024^3 float32, 1024 uniform thresholds,
    device-resident input (4 GiB > L2), CUDA-event timing over K steps,
    gated bit-exact against the oracle (accumulated slab by slab)."""
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
    h = hist.cpu().numpy().reshape(-1)
    _gate(int(h.sum()) == 1 and int(curve.reshape(-1)[-1]) == 1, "NS sum of coefficients")
    parity = "invariants only"
    if not args.no_parity:
        from oracle import parity as OP

        _gate(np.array_equal(h, OP.counter_slab_hist(SEED + 1, (n, n, n), 0, n, taus.taus, slab=128)),
              "NS histogram vs oracle")
        parity = "checked: bit-exact vs the CPU oracle on the timed 1024^3 volume"
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
    e2e = None
    if not args.no_e2e:
        # the 4 GiB volume pinned host -> HBM in 64-plane chunks through
        # ecc_discrete_host (the planes on the device are deposited while the
        # next chunk is copied), curve -> host
        host = torch.empty(x.shape, dtype=torch.float32, pin_memory=True)
        host.copy_(x.cpu())
        want = curve.cpu().numpy().reshape(-1)
        got = E.ecc_discrete_host(host, taus, chunk_planes=64).cpu().numpy().reshape(-1)
        _gate(np.array_equal(got, want), "NS e2e curve")
        t0 = time.perf_counter()
        for _ in range(2):
            E.ecc_discrete_host(host, taus, chunk_planes=64).cpu()
        e_ms = (time.perf_counter() - t0) * 1e3 / 2
        e2e = {"value": x.numel() / (e_ms * 1e-3) / 1e9, "unit": UNIT, "ms_per_step": e_ms,
               "h2d_bytes_per_step": int(host.numel() * 4), "d2h_bytes_per_step": NB * 8,
               "api": "paper_2510_20271_b200.ecc_discrete_host (64-plane chunks, pinned host -> HBM inside the "
                      "timed region)"}
        del host
    cpu = None
    if not args.no_cpu:
        # the CPU port on a bounded sample of the same workload: 64 planes of
        # 1024 x 1024 (all host threads), per-voxel rate
        from oracle import oracle

        oracle.set_threads(os.cpu_count() or 1)
        xs = oracle.counter_grid(SEED + 1, (64, n, n)).reshape(64, n, n)
        t0 = time.perf_counter()
        oracle.histogram(xs, taus.taus)
        v_cpu = xs.size / (time.perf_counter() - t0) / 1e9
        cpu = {"value": v_cpu, "unit": UNIT, "cores": os.cpu_count() or 1, "kind": "port",
               "sample": f"64 planes of the 1024^2 NS counter volume, {NB} bins, all host threads (per-voxel rate)",
               "extrapolated_ms_per_step": x.numel() / (v_cpu * 1e9) * 1e3}
        del xs
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
           "parity": parity, "e2e": e2e, "cpu_baseline": cpu,
           "roofline": {"bound": "hbm", "achieved": gbs, "peak": peak, "unit": "GB/s", "frac": gbs / peak,
                        "peak_source": peak_kind, "traffic": traffic,
                        "algorithmic_bytes_per_launch": 4 * x.numel()}}
    del x, curve, hist
    torch.cuda.empty_cache()
    return out


def bench_c5(args, dev, world, rank, dist_on=False):
    """C5: the 2048^3 float32 counter volume cut into N z-slabs, one per GPU
    (strong scaling: the total volume is fixed).  A step is the distributed
    pipeline: halo exchange with the z-neighbours, the fused slab sweep
    (ecc_histogram_range, one launch over the own planes), the NCCL
    all-reduce of the (B+1) int64 histogram and the scan.  1024 thresholds
    uniform over the generator's range.  Gate: the sum invariant of the whole
    volume, and the kernel bit-exact vs the oracle on the slab's first 64
    planes taken as a volume of C5's 2048 x 2048 planes."""
    import torch
    import torch.distributed as dist

    import paper_2510_20271_b200 as E
    from paper_2510_20271_b200 import _lib
    from paper_2510_20271_b200 import distributed as D

    L = _lib.lib()
    Dz, H, W = args.c5_depth, 2048, 2048
    if dist_on:
        z0, z1 = D.slab_bounds(Dz, world, rank)
    else:
        z0, z1 = 0, Dz
    P = z1 - z0
    padded = D.alloc_padded_slab(P, (H, W), torch.float32, dev)
    lo_plane = max(z0 - 1, 0)
    hi_plane = min(z1 + 1, Dz)
    first = 1 - (z0 - lo_plane)
    gen = padded[first:first + (hi_plane - lo_plane)]
    _lib.check(L.ecc_counter_grid(SEED + 2, lo_plane * H * W, gen.numel(), _lib.ptr(gen), _lib.stream_ptr(gen)))
    taus = E.thresholds_from_range(0.0, 1.0 - 2.0 ** -24, NB)
    table, binning = taus.device_table(_lib.DTYPE_F32, dev)
    stream = torch.cuda.current_stream(dev)
    curve = torch.empty(NB, dtype=torch.int64, device=dev)
    dims_cache = {}

    def slab_fn(v, a, b, t):
        out = torch.empty(NB + 1, dtype=torch.int64, device=dev)
        dv = dims_cache.get(tuple(v.shape))
        if dv is None:
            dv = dims_cache[tuple(v.shape)] = _lib.dims_arg(v.shape)
        _lib.check(L.ecc_histogram_range(_lib.ptr(v), _lib.DTYPE_F32, 3, _lib.ptr(dv), 1, a, b, _lib.ptr(table),
                                         _lib.ctypes.byref(binning), _lib.ptr(out),
                                         _lib.ctypes.c_void_p(stream.cuda_stream)))
        return out

    whole = padded[1:-1]

    def step():
        if dist_on:
            h = D.slab_histogram(padded, taus, hist_fn=slab_fn, depth=Dz)
        else:
            h = slab_fn(whole, 0, P, taus)
        _lib.check(L.ecc_scan(_lib.ptr(h), 1, NB, _lib.ptr(curve), _lib.ctypes.c_void_p(stream.cuda_stream)))
        return h

    h = step().cpu().numpy()
    _gate(int(h.sum()) == 1, "C5 sum of coefficients")
    parity = "invariants only"
    if rank == 0 and not args.no_parity:
        from oracle import parity as OP

        k = min(64, P)
        sub = whole[:k].contiguous()
        got = E.histogram_device(sub, taus).cpu().numpy().reshape(-1)
        want = OP.counter_slab_hist(SEED + 2, (k, H, W), 0, k, taus.taus, slab=32) if z0 == 0 else None
        if want is not None:
            _gate(np.array_equal(got, want), "C5 kernel on 64 planes of 2048^2 vs oracle")
            parity = ("checked: global sum invariant; the kernel bit-exact vs the CPU oracle on the first "
                      f"{k} planes of the C5 volume taken as a volume")
        del sub
    if dist_on:
        dist.barrier(device_ids=[dev.index])
    for _ in range(2):
        step()
    torch.cuda.synchronize()
    if dist_on:
        dist.barrier(device_ids=[dev.index])
    steps = max(3, min(args.steps, 10))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = _max_over_ranks([e0.elapsed_time(e1) / steps], dev, dist_on)[0]
    peak, peak_kind = _peaks()
    vox = Dz * H * W
    gbs_gpu = 4.0 * vox / world / (ms * 1e-3) / 1e9
    out = {"workload": f"C5: 3D {Dz}x2048x2048 float32 counter volume, discrete ECC, 1024 thresholds, "
                       f"z-slabs over {world} GPU(s): halo exchange + slab sweep + NCCL histogram all-reduce",
           "value": vox / (ms * 1e-3) / 1e9, "unit": UNIT, "ms_per_step": ms, "steps": steps,
           "n_gpus": world, "scaling": "strong", "planes_per_gpu": P, "parity": parity,
           "gpu_launches_per_step": 2,
           "roofline": {"bound": "hbm", "achieved": gbs_gpu, "peak": peak, "unit": "GB/s",
                        "frac": gbs_gpu / peak, "peak_source": peak_kind, "per": "GPU"},
           "e2e": None}
    # e2e: the rank's slab from pinned host memory through the public API
    # every step (N = 1: ecc_discrete_host streams the 32 GiB volume through
    # device ring buffers; N > 1: the slab copied into the padded buffer, then
    # distributed.slab_curve), the curve back to the host.  Needs the slab in
    # pinned host memory: skipped when the host lacks room for it.
    if not args.no_e2e:
        slab_bytes = 4 * P * H * W
        try:
            import psutil

            avail = psutil.virtual_memory().available
        except Exception:   # noqa: BLE001
            avail = 0
        ok_all = torch.tensor([1 if avail >= 3 * slab_bytes else 0], device=dev)
        if dist_on:
            dist.all_reduce(ok_all, op=dist.ReduceOp.MIN)
        if int(ok_all.item()):
            want_curve = curve.cpu()
            host = torch.empty((P, H, W), dtype=torch.float32, pin_memory=True)
            host.copy_(whole)
            if not dist_on:
                def e2e_step():
                    return E.ecc_discrete_host(host, taus, chunk_planes=64).cpu()
                api = ("paper_2510_20271_b200.ecc_discrete_host (the 32 GiB volume streamed from pinned host memory "
                       "through device ring buffers of 64-plane chunks)")
            else:
                def e2e_step():
                    padded[1:-1].copy_(host, non_blocking=True)
                    return D.slab_curve(padded, taus, depth=Dz).cpu()
                api = ("paper_2510_20271_b200.distributed.slab_curve (the rank's slab copied pinned host -> HBM, "
                       "halo exchange, slab sweep, NCCL all-reduce, scan)")
            got = e2e_step()
            _gate(np.array_equal(got.numpy(), want_curve.numpy()), "C5 e2e curve")
            if dist_on:
                dist.barrier(device_ids=[dev.index])
            t0 = time.perf_counter()
            reps = 2
            for _ in range(reps):
                e2e_step()
            torch.cuda.synchronize()
            e_ms = _max_over_ranks([(time.perf_counter() - t0) * 1e3 / reps], dev, dist_on)[0]
            out["e2e"] = {"value": vox / (e_ms * 1e-3) / 1e9, "unit": UNIT, "ms_per_step": e_ms,
                          "h2d_bytes_per_step": 4 * vox, "d2h_bytes_per_step": NB * 8 * world,
                          "api": api + " (pinned host -> HBM copy inside the timed region)"}
            del host
        else:
            out["e2e_note"] = (f"not measured: the host lacks room to pin this rank's {slab_bytes / 2 ** 30:.0f} GiB "
                               "slab (3x its size must be available)")
    del padded, gen, whole
    torch.cuda.empty_cache()
    if rank == 0 and not args.no_cpu:
        # the CPU port on a bounded sample of the same workload: 16 planes of
        # 2048 x 2048 (all host threads), per-voxel rate
        from oracle import oracle

        oracle.set_threads(os.cpu_count() or 1)
        xs = oracle.counter_grid(SEED + 2, (16, H, W)).reshape(16, H, W)
        t0 = time.perf_counter()
        oracle.histogram(xs, np.linspace(0.0, 1.0 - 2.0 ** -24, NB))
        v_cpu = xs.size / (time.perf_counter() - t0) / 1e9
        out["cpu_baseline"] = {"value": v_cpu, "unit": UNIT, "cores": os.cpu_count() or 1, "kind": "port",
                               "sample": f"16 planes of the 2048^2 C5 counter volume, {NB} bins, all host threads "
                                         "(per-voxel rate)",
                               "extrapolated_ms_per_step": vox / (v_cpu * 1e9) * 1e3}
        del xs
    return out


def _soft_pipe_ops(nz: float, vox: int, B: int, win: int):
    """(MUFU ops, FMA-pipe lane ops) the soft kernels issue per fwd+bwd step.
    Band kernels (win < B): only c != 0 voxels and the window's pairs; the
    forward pairs every two reciprocals (0.5 MUFU + 3.5 lane-FMA per pair),
    the backward keeps half of its slot pairs unpaired (0.75 MUFU + 4.75
    lane-FMA per pair); one ex2 per voxel and lane (1/16 per pair).  Full
    kernels: all B thresholds, forward paired, backward 7/8 of the pairs on
    MUFU (ecc_soft.cu)."""
    if win < B:
        pairs = nz * vox * win
        return pairs * ((0.5 + 1.0 / 16.0) + (0.75 + 1.0 / 16.0)), pairs * (3.5 + 4.75)
    pairs = nz * vox * B
    return pairs * ((0.5 + 1.0 / 16.0) + (7.0 / 8.0 + 1.0 / 16.0)), pairs * (3.5 + 5.0)


def _soft_setup(ndim: int):
    B, lam, alpha = 256, 50.0, 0.3
    v = np.array([1.0, 2.0]) if ndim == 2 else np.array([1.0, 2.0, -0.5])
    u = v / np.linalg.norm(v)
    span = alpha * np.abs(u).sum()
    return B, lam, alpha, v, u, np.linspace(-span, 1.0 + span, B + 1)[1:]


def _soft_gate(E, x_np, taus, v, alpha, lam, dev, what):
    """Module forward + backward on x_np (a few images / one small volume)
    against the oracle: chi, d_values, d_tau, d_v, d_alpha normwise <= 1e-4."""
    import torch

    from oracle import parity as OP

    m = E.SoftECC(taus, v, alpha=alpha, lam=lam).to(dev)
    xt = torch.from_numpy(x_np).to(dev).requires_grad_(True)
    chi = m(xt)
    rng = np.random.default_rng(7)
    up = rng.uniform(0.5, 1.5, (x_np.shape[0], len(taus)))
    (chi * torch.from_numpy(up).to(dev)).sum().backward()
    u = v / np.linalg.norm(v)
    gtau, G = np.zeros(len(taus)), np.zeros(len(v))
    worst = 0.0

    def nw(a, b):
        return float(np.abs(np.asarray(a, np.float64) - b).max() / max(np.abs(b).max(), 1e-300))

    for i in range(x_np.shape[0]):
        c_chi, dv, dt, _, _, Gi = OP.soft_item(x_np[i], lam, alpha, u, taus, up[i])
        worst = max(worst, nw(chi[i].detach().cpu().numpy(), c_chi), nw(xt.grad[i].cpu().numpy(), dv))
        gtau += dt
        G += Gi
    worst = max(worst, nw(m.taus.grad.cpu().numpy(), gtau))
    du_raw = -alpha * G
    worst = max(worst, nw(m.v.grad.cpu().numpy(), (du_raw - u * (u @ du_raw)) / np.linalg.norm(v)))
    da = -(G @ u)
    worst = max(worst, abs(float(m.alpha.grad) - da) / max(abs(da), 1e-4))
    _gate(worst <= 1e-4, f"{what}: normwise error {worst:.2e} > 1e-4")
    return worst


def bench_c4(args, dev, world, rank, dist_on=False):
    """C4: 3D 1024^3 float32 soft ECC, forward + backward, learnable tau / v /
    alpha, batch-sharded (one item per GPU), B = 256, lambda = 50, alpha =
    0.3, u = normalize(1, 2, -0.5); the shared parameters'
    gradients are all-reduced under torchrun (distributed.allreduce_soft_grads)."""
    import torch

    import paper_2510_20271_b200 as E

    n = 1024
    B, lam, alpha, v, u, taus0 = _soft_setup(3)
    g = torch.Generator(device=dev)
    g.manual_seed(SEED + 100 + rank)
    x = torch.rand((1, n, n, n), device=dev, generator=g, dtype=torch.float32)
    m = E.SoftECC(taus0, v, alpha=alpha, lam=lam).to(dev)
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
    ms = _max_over_ranks([e0.elapsed_time(e1) / steps], dev, dist_on)[0]
    _gate(bool(torch.isfinite(m.taus.grad).all()) and bool(torch.isfinite(m.v.grad).all()), "C4 finite gradients")
    # MUFU work issued (as the C3 leg): c != 0 voxels only, the band window
    from paper_2510_20271_b200 import soft as S
    from paper_2510_20271_b200.soft import band_window

    p = S._params(lam, alpha, u, float(taus0[0]), float(taus0[-1]), 3, S._block_halfwidth(taus0))
    c0, _ = S.soft_prepare_device(x[:, :128].contiguous(), (128, n, n), 1, p)
    nz = float(torch.count_nonzero(c0)) / c0.numel()
    del c0
    win = band_window(taus0, lam)
    # e2e through soft_step_host: the item pinned host -> HBM (streamed in
    # z-slabs under the prepare, forward and backward of the resident
    # planes), chi and the parameter gradients -> host
    e2e = None
    if not args.no_e2e:
        host = torch.empty(x.shape, dtype=torch.float32, pin_memory=True)
        host.copy_(x.cpu())

        def e2e_step():
            m.zero_grad(set_to_none=True)
            chi = E.soft_step_host(m, host, up, micro=1)
            if dist_on:
                from paper_2510_20271_b200 import distributed as D

                D.allreduce_soft_grads(m)
            return (chi.cpu(), m.taus.grad.cpu(), m.v.grad.cpu(), m.alpha.grad.cpu())

        e2e_step()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(2):
            e2e_step()
        torch.cuda.synchronize()
        e_ms = _max_over_ranks([(time.perf_counter() - t0) * 1e3 / 2], dev, dist_on)[0]
        e2e = {"value": n ** 3 * world / (e_ms * 1e-3), "unit": "voxel/s", "ms_per_step": e_ms,
               "h2d_bytes_per_step": int(host.numel() * 4) * world,
               "d2h_bytes_per_step": (B * 8 + B * 8 + 3 * 8 + 8) * world,
               "api": "paper_2510_20271_b200.soft_step_host (the 1024^3 item pinned host -> HBM in z-slabs of 16 "
                      "planes; the prepare, forward and backward of the resident planes overlap the rest of the "
                      "copy; chi and the tau / v / alpha gradients -> host, inside the timed region)"}
        del host
    del x, m
    torch.cuda.empty_cache()
    parity = "finite gradients only"
    if rank == 0 and not args.no_parity:
        rng = np.random.default_rng(SEED + 100)
        err = _soft_gate(E, rng.random((1, 128, 128, 128)).astype(np.float32), taus0, v, alpha, lam, dev,
                         "C4 module on 128^3")
        parity = (f"checked: the same 3-D module path on a 128^3 volume vs the CPU oracle (max normwise "
                  f"error {err:.1e} <= 1e-4); the timed 1024^3 item: finite gradients")
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        v_s, cores, sample, nvox = cpu_soft_sample(3)
        cpu = {"value": v_s, "unit": "voxel/s", "cores": cores, "kind": "port",
               "sample": sample, "extrapolated_ms_per_step": n ** 3 / v_s * 1e3}
    vox = n ** 3 * world
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    mufu_peak = 16 * sms * 1.965e9 * world
    mufu_ops, fma_ops = _soft_pipe_ops(nz, vox, B, win)
    fma_peak = 116.5 * sms * 1.965e9 * world   # FFMA lane-ops/s (tools/microbench/pipes.cu)
    return {"workload": "C4: 3D 1024^3 float32 soft ECC fwd+bwd, learnable tau/u/alpha, one item per GPU",
            "value": vox / (ms * 1e-3), "unit": "voxel/s", "ms_per_step": ms, "steps": steps,
            "n_gpus": world, "bins": B, "lambda": lam, "alpha": alpha, "parallelism": f"batch{world}",
            "scaling": "weak", "parity": parity, "cpu_baseline": cpu, "e2e": e2e,
            "roofline": {"bound": "sfu", "unit": "MUFU ops/s", "achieved": mufu_ops / (ms * 1e-3),
                         "peak": mufu_peak, "frac": mufu_ops / (ms * 1e-3) / mufu_peak,
                         "nonzero_fraction": nz, "window_thresholds": win,
                         "fma_pipe_frac": fma_ops / (ms * 1e-3) / fma_peak,
                         "algorithmic_pairs_per_s": 2 * vox * B / (ms * 1e-3),
                         "survey_sfu_bound_voxel_s": mufu_peak / (2 * B),
                         "peak_source": "MUFU.RCP 15.9 lane-ops/SM-clk (tools/microbench/pipes.cu) x SMs x 1.965 GHz"},
            "algorithmic_pairs_per_s": 2 * vox * B / (ms * 1e-3)}


def bench_soft(args, dev, world, rank, dist_on=False):
    import torch

    import paper_2510_20271_b200 as E

    N, H, W = args.soft_batch, 1024, 1024
    B, lam, alpha, v, u, taus = _soft_setup(2)
    g = torch.Generator(device=dev)
    g.manual_seed(SEED + rank)
    x = torch.rand((N, H, W), device=dev, generator=g, dtype=torch.float32)
    m = E.SoftECC(taus, v, alpha=alpha, lam=lam).to(dev)
    up = torch.ones((N, B), dtype=torch.float64, device=dev)

    def step(xx):
        m.zero_grad(set_to_none=True)
        chi = m(xx)
        chi.backward(up)
        if dist_on:
            from paper_2510_20271_b200 import distributed as D

            D.allreduce_soft_grads(m)
        return chi

    step(x)
    torch.cuda.synchronize()
    steps = max(2, min(args.steps, 5))
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        step(x)
    e1.record()
    torch.cuda.synchronize()
    ms = _max_over_ranks([e0.elapsed_time(e1) / steps], dev, dist_on)[0]
    # fraction of voxels with c != 0 (the kernels skip the others)
    from paper_2510_20271_b200 import soft as S

    p = S._params(lam, alpha, u, float(taus[0]), float(taus[-1]), 2, S._block_halfwidth(taus))
    c0, _ = S.soft_prepare_device(x[:8].contiguous(), (H, W), min(N, 8), p)
    nz = float(torch.count_nonzero(c0)) / c0.numel()
    del c0

    # e2e through the module: each step copies the batch pinned host -> HBM,
    # runs forward + backward, and reads chi and the parameter gradients back
    e2e = None
    if not args.no_e2e:
        host = torch.empty((N, H, W), dtype=torch.float32, pin_memory=True)
        host.copy_(x.cpu())

        def e2e_step():
            # groups of 4 images: the next group's copy overlaps this group's
            # prepare, forward and backward (soft_step_host)
            m.zero_grad(set_to_none=True)
            chi = E.soft_step_host(m, host, up, micro=4)
            if dist_on:
                from paper_2510_20271_b200 import distributed as D

                D.allreduce_soft_grads(m)
            return (chi.cpu(), m.taus.grad.cpu(), m.v.grad.cpu(), m.alpha.grad.cpu())

        e2e_step()
        torch.cuda.synchronize()
        reps = max(2, min(args.steps, 5))
        t0 = time.perf_counter()
        for _ in range(reps):
            e2e_step()
        torch.cuda.synchronize()
        e_ms = _max_over_ranks([(time.perf_counter() - t0) * 1e3 / reps], dev, dist_on)[0]
        e2e = {"value": N * H * W * world / (e_ms * 1e-3), "unit": "voxel/s", "ms_per_step": e_ms,
               "h2d_bytes_per_step": int(host.numel() * 4) * world,
               "d2h_bytes_per_step": (N * B * 8 + B * 8 + 2 * 8 + 8) * world,
               "api": "paper_2510_20271_b200.soft_step_host: the batch copied pinned host -> HBM in groups of 4 "
                      "images, each group's prepare, forward and backward running while the next is copied; chi "
                      "and the tau / v / alpha gradients -> host, inside the timed region"}
        del host
    del x
    torch.cuda.empty_cache()
    parity = "not checked"
    if rank == 0 and not args.no_parity:
        rng = np.random.default_rng(SEED)
        err = _soft_gate(E, rng.random((2, H, W)).astype(np.float32), taus, v, alpha, lam, dev,
                         "C3 module on 2 full images")
        parity = (f"checked: the same module path on 2 full 1024x1024 images vs the CPU oracle "
                  f"(chi, d_values, d_tau, d_v, d_alpha; max normwise error {err:.1e} <= 1e-4)")
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        v_s, cores, sample, _ = cpu_soft_sample(2)
        cpu = {"value": v_s, "unit": "voxel/s", "cores": cores, "kind": "port", "sample": sample,
               "extrapolated_ms_per_step": N * H * W / v_s * 1e3}
    vox = N * H * W * world
    pairs = vox * B * 2                      # algorithmic (voxel, threshold) pairs, forward + backward
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    mufu_peak = 16 * sms * 1.965e9 * world   # MUFU.RCP lane-ops/s (15.9/clk/SM measured, tools/microbench)
    # MUFU and FMA-pipe work actually issued (_soft_pipe_ops): the kernels
    # evaluate only c != 0 voxels, and with the band kernels only a window of
    # `win` thresholds per voxel (the saturated pairs outside it are exact
    # 0 / 1 to 2^-24)
    from paper_2510_20271_b200.soft import band_window

    win = band_window(taus, lam)
    mufu_ops, fma_ops = _soft_pipe_ops(nz, vox, B, win)
    fma_peak = 116.5 * sms * 1.965e9 * world   # FFMA lane-ops/s (tools/microbench/pipes.cu)
    return {"metric": "soft-ECC fwd+bwd voxels/s", "value": vox / (ms * 1e-3), "unit": "voxel/s",
            "ms_per_step": ms, "steps": steps, "parity": parity, "cpu_baseline": cpu, "e2e": e2e,
            "config": {"workload": "C3: batched 2D 128x1024x1024 f32, soft ECC fwd+bwd, learnable tau/u/alpha",
                       "batch_per_gpu": N, "bins": B, "lambda": lam, "alpha": alpha, "parallelism": f"batch{world}"},
            "roofline": {"bound": "sfu", "unit": "MUFU ops/s", "achieved": mufu_ops / (ms * 1e-3),
                         "peak": mufu_peak, "frac": mufu_ops / (ms * 1e-3) / mufu_peak,
                         "nonzero_fraction": nz, "algorithmic_pairs_per_s": pairs / (ms * 1e-3),
                         "window_thresholds": win, "fma_pipe_frac": fma_ops / (ms * 1e-3) / fma_peak,
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
    ap.add_argument("--c5-depth", type=int, default=2048, help="planes of the C5 volume (2048 = C5)")
    ap.add_argument("--soft-batch", type=int, default=128)
    ap.add_argument("--no-soft", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-parity", action="store_true", help="skip the oracle gates (invariants only)")
    ap.add_argument("--no-ns", action="store_true", help="skip the 1024^3 north-star measurement")
    ap.add_argument("--no-c4", action="store_true", help="skip the 1024^3 soft (C4) measurement")
    ap.add_argument("--no-c5", action="store_true", help="skip the C5 2048^3 measurement")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()

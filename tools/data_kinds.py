"""The rank4 sweep on the synthetic input kinds of SURVEY §8(d) (development
aid): uniform counter values (the bench input), gaussian blobs (smooth: most
c = 0 and long runs of equal ranks, i.e. the hot-counter pattern for the
shared-memory atomics) and a radial gradient, 512^3 and 1024^3 f32, 1024
uniform thresholds over the grid's range; device time of back-to-back
launches, and the histogram checked bit for bit against the CPU oracle
(slab-wise rows).

    python tools/data_kinds.py [n ...]
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2510_20271_b200 as E  # noqa: E402
from paper_2510_20271_b200 import _lib  # noqa: E402
from oracle import oracle  # noqa: E402   (checker only)


def blobs(n, seed=0, count=8):
    # synthetic.py's gaussian-blobs formula, evaluated on the device in float64
    rng = np.random.default_rng(seed)
    width = max(n / 8.0, 1.0)
    centres = rng.uniform(0, 1, size=(count, 3)) * (n - 1)
    ax = torch.arange(n, device="cuda", dtype=torch.float64)
    acc = torch.zeros((n, n, n), device="cuda", dtype=torch.float64)
    for c in centres:
        gz = torch.exp(-(ax - c[0]) ** 2 / (2 * width ** 2))
        gy = torch.exp(-(ax - c[1]) ** 2 / (2 * width ** 2))
        gx = torch.exp(-(ax - c[2]) ** 2 / (2 * width ** 2))
        acc += gz[:, None, None] * gy[None, :, None] * gx[None, None, :]
    return (acc / acc.max()).float()


def radial(n):
    ax = torch.arange(n, device="cuda", dtype=torch.float64) - (n - 1) / 2
    r2 = ax[:, None, None] ** 2 + ax[None, :, None] ** 2 + ax[None, None, :] ** 2
    return (torch.sqrt(r2) / np.sqrt(3 * ((n - 1) / 2) ** 2)).float()


def counter(n):
    x = torch.empty((n, n, n), device="cuda")
    _lib.check(_lib.lib().ecc_counter_grid(11, 0, x.numel(), _lib.ptr(x), _lib.stream_ptr(x)))
    return x


def timed(x, ts):
    for _ in range(3):
        E.histogram_device(x, ts)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(10):
            E.histogram_device(x, ts)
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e) / 10)
    return best


import os  # noqa: E402

sizes = [int(a) for a in sys.argv[1:]] or [512, 1024]
only = os.environ.get("KINDS", "counter,gaussian-blobs,radial-gradient").split(",")
for n in sizes:
    for kind, gen in (("counter", counter), ("gaussian-blobs", blobs), ("radial-gradient", radial)):
        if kind not in only:
            continue
        x = gen(n)
        lo, hi = float(x.min()), float(x.max())
        ts = E.thresholds_from_range(lo, hi, 1024)
        ms = timed(x, ts)
        h = E.histogram_device(x, ts).cpu().numpy().reshape(-1)
        # parity: the oracle's histogram, 32 planes at a time (bounded host memory)
        ok = None
        if not os.environ.get("NOPARITY"):
            xh = x.cpu().numpy()
            want = np.zeros(ts.taus.size + 1, np.int64)
            for z in range(0, n, 32):
                want += oracle.histogram_rows(xh, z, min(n, z + 32), ts.taus)
            ok = np.array_equal(h, want)
            del xh
        print(f"{kind:16s} {n}^3: {ms * 1e3:8.1f} us  {n ** 3 / ms / 1e6:6.1f} Gvox/s  "
              f"{4 * n ** 3 / ms / 1e6 / 6535.1:.3f} of HBM  bit-exact vs oracle: {ok}", flush=True)
        del x
        torch.cuda.empty_cache()

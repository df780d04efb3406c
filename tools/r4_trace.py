"""Per-CTA timeline of one rank4 launch (development aid): needs a library built
with -DECC_R4_TRACE (python tools/variants.py trace="-DECC_R4_TRACE") and
ECC_B200_LIB=tools/_v/trace.so.  Prints the ramp (launch -> first plane ranked),
the spread of the CTAs' loop ends, the flush and the per-SM idle tail.

    ECC_B200_LIB=tools/_v/trace.so python tools/r4_trace.py 512 [1024 ...]
"""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2510_20271_b200 as E
from paper_2510_20271_b200 import _lib

L = _lib.lib()
L.ecc_r4_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
ts = E.thresholds_from_range(0.0, 1.0, 1024)
for n in [int(a) for a in sys.argv[1:]] or [512]:
    x = torch.empty((n, n, n), device="cuda")
    _lib.check(L.ecc_counter_grid(11, 0, x.numel(), _lib.ptr(x), _lib.stream_ptr(x)))
    for _ in range(5):
        E.histogram_device(x, ts)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(10):
            h = E.histogram_device(x, ts)
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e) / 10)
    import hashlib
    print(f"{n}^3: back-to-back {best * 1e3:.1f} us/launch ({n ** 3 / best / 1e6:.1f} Gvox/s), "
          f"result sha {hashlib.sha256(h.cpu().numpy().tobytes()).hexdigest()[:12]}")
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    E.histogram_device(x, ts)
    e.record()
    torch.cuda.synchronize()
    buf = np.zeros(8 * 8192, np.uint64)
    assert L.ecc_r4_trace_read(buf.ctypes.data, buf.nbytes) == 0
    t = buf.reshape(8192, 8).astype(np.int64)
    t = t[t[:, 1] > 0]
    t = t[t[:, 1] >= t[:, 1].max() - 10_000_000]   # this launch only (10 ms window)
    t0 = t[:, 1].min()
    sm = t[:, 0]
    start = (t[:, 1] - t0) / 1e3
    first = (t[:, 2] - t0) / 1e3
    wend = (t[:, 3:7] - t0) / 1e3
    fend = (t[:, 7] - t0) / 1e3
    lend = wend.max(1)
    T = fend.max()
    print(f"\n{n}^3: {len(t)} CTAs, event time {s.elapsed_time(e) * 1e3:.1f} us, trace span {T:.1f} us")
    q = lambda a: " ".join(f"{v:6.1f}" for v in np.percentile(a, [0, 10, 50, 90, 100]))
    print(f"  CTA start          (min p10 p50 p90 max) {q(start)}")
    print(f"  first plane ranked - start                {q(first - start)}")
    print(f"  loop end (last warp)                      {q(lend)}")
    print(f"  warp spread in CTA (last - first warp)    {q(wend.max(1) - wend.min(1))}")
    print(f"  flush (end - last warp)                   {q(fend - lend)}")
    print(f"  CTA end                                   {q(fend)}")
    # per-SM busy fraction: resident CTAs over time (each CTA occupies [start, fend])
    grid = np.linspace(0, T, 400)
    occ = np.zeros((int(sm.max()) + 1, grid.size))
    for i in range(len(t)):
        occ[sm[i]] += (grid >= start[i]) & (grid < fend[i])
    used = occ[occ.sum(1) > 0]
    mean_res = used.mean(0)
    print(f"  mean resident CTAs per SM over time (10 slices): "
          + " ".join(f"{v:.2f}" for v in mean_res.reshape(10, -1).mean(1)))
    bid = np.nonzero(buf.reshape(8192, 8)[:, 1] > 0)[0][: len(t)]
    print("  SM of blocks 0..23:", " ".join(str(v) for v in sm[:24]))
    # SM-local rank of each CTA by block index (the dispatch order)
    loc = np.zeros(len(t), int)
    for k in np.unique(sm):
        idx = np.nonzero(sm == k)[0]
        loc[idx[np.argsort(bid[idx])]] = np.arange(idx.size)
    for r in range(loc.max() + 1):
        m = loc == r
        print(f"  SM-local rank {r}: {m.sum():4d} CTAs, loop end {q(lend[m])}")
    last_sm_end = np.array([fend[sm == k].max() for k in np.unique(sm)])
    print(f"  per-SM last CTA end                       {q(last_sm_end)}")
    del x
    torch.cuda.empty_cache()

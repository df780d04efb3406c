"""A/B device timings of kernel variants (f3 variants, ecc_set_variant) on the C2/NS volumes;
every variant's histogram must equal the first one's (development aid)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2510_20271_b200 as E
from paper_2510_20271_b200 import _lib

variants = sys.argv[1].split(",") if len(sys.argv) > 1 else ["", "edge1"]
sizes = [int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else [512, 1024]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
for n in sizes:
    x = torch.empty((n, n, n), dtype=torch.float32, device="cuda")
    _lib.check(_lib.lib().ecc_counter_grid(11, 0, x.numel(), _lib.ptr(x), _lib.stream_ptr(x)))
    lo, hi, _ = E.device_minmax(x)
    ts = E.thresholds_from_range(lo, hi, 1024)
    ref = None
    res = {}
    for rnd in range(2):
        for v in variants:
            _lib.set_variant("f3", v or "default")
            h = E.histogram_device(x, ts).cpu().numpy()
            if ref is None:
                ref = h
            assert np.array_equal(h, ref), f"variant {v!r} differs at {n}^3"
            for _ in range(3):
                E.histogram_device(x, ts)
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ts_ = []
            for _ in range(reps):
                s.record(); E.histogram_device(x, ts); e.record(); torch.cuda.synchronize()
                ts_.append(s.elapsed_time(e))
            res.setdefault(v, []).append(float(np.median(ts_)))
    for v, t in res.items():
        ms = min(t)
        print(f"{n}^3 {v or 'default':10s} {ms:.4f} ms  {x.numel()/ms/1e6:7.1f} Gvox/s  frac {4*x.numel()/ms/1e6/6535.1:.3f}", flush=True)
    del x
    torch.cuda.empty_cache()

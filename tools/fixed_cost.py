"""Fixed (per-launch) vs per-plane cost of the 512^2-plane rank4 sweep: device time at several depths
and a linear fit (development aid)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2510_20271_b200 as E
from paper_2510_20271_b200 import _lib

ts = E.thresholds_from_range(0.0, 1.0, 1024)
rows = []
for d in (64, 128, 256, 384, 512, 768, 1024):
    x = torch.empty((d, 512, 512), device="cuda")
    _lib.check(_lib.lib().ecc_counter_grid(11, 0, x.numel(), _lib.ptr(x), _lib.stream_ptr(x)))
    for _ in range(3):
        E.histogram_device(x, ts)
    torch.cuda.synchronize()
    best = 1e9
    for r in range(5):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(10):
            E.histogram_device(x, ts)
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e) / 10)
    rows.append((d, best))
    print(f"{d:5d} planes: {best * 1e3:8.1f} us  {d * 512 * 512 / best / 1e6:6.1f} Gvox/s", flush=True)
    del x
    torch.cuda.empty_cache()
d = np.array([r[0] for r in rows], float)
t = np.array([r[1] for r in rows]) * 1e3
A = np.vstack([np.ones_like(d), d]).T
(a, b), *_ = np.linalg.lstsq(A, t, rcond=None)
print(f"fit: {a:.1f} us + {b:.3f} us/plane")

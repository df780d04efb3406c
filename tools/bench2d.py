"""Batched 2D discrete ECC timing (development aid)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2510_20271_b200 as E
from paper_2510_20271_b200 import _lib

N, H, W = (int(a) for a in (sys.argv[1:4] if len(sys.argv) > 3 else (128, 1024, 1024)))
x = torch.empty((N, H, W), dtype=torch.float32, device="cuda")
_lib.check(_lib.lib().ecc_counter_grid(5, 0, x.numel(), _lib.ptr(x), _lib.stream_ptr(x)))
ts = E.thresholds_from_range(0.0, 1.0, 1024)
for _ in range(3):
    E.ecc_discrete(x, ts, ndim=2)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(5):
    E.histogram_device(x, ts, ndim=2)
e.record(); torch.cuda.synchronize()
ms = s.elapsed_time(e) / 5
print(f"2D {N}x{H}x{W} B=1024: {ms:.3f} ms  {x.numel() / ms / 1e6:.1f} Gvox/s")

"""Discrete ECC timing over volume shapes (development aid)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2510_20271_b200 as E
from paper_2510_20271_b200 import _lib

def timeit(fn, reps=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps

shapes = [(128, 512, 512), (256, 512, 512), (512, 512, 512), (1024, 512, 512), (2048, 512, 512),
          (512, 1024, 1024), (256, 2048, 2048), (1024, 1024, 1024)]
ts = E.thresholds_from_range(0.0, 1.0 - 2 ** -24, 1024)
for sh in shapes:
    x = torch.empty(sh, dtype=torch.float32, device="cuda")
    _lib.check(_lib.lib().ecc_counter_grid(11, 0, x.numel(), _lib.ptr(x), _lib.stream_ptr(x)))
    ms = timeit(lambda: E.histogram_device(x, ts))
    print(f"{'x'.join(map(str, sh)):>16}: {ms:.3f} ms  {x.numel() / ms / 1e6:.1f} Gvox/s", flush=True)
    del x

"""A shallow 512^2-plane volume through the rank4 kernel (profiling target for the per-launch fixed cost)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2510_20271_b200 as E
from paper_2510_20271_b200 import _lib

d = int(sys.argv[1]) if len(sys.argv) > 1 else 64
x = torch.empty((d, 512, 512), dtype=torch.float32, device="cuda")
_lib.check(_lib.lib().ecc_counter_grid(11, 0, x.numel(), _lib.ptr(x), _lib.stream_ptr(x)))
ts = E.thresholds_from_range(0.0, 1.0, 1024)
for _ in range(3):
    E.histogram_device(x, ts)
torch.cuda.synchronize()
print("ok")

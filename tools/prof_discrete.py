"""Run the discrete hot kernel a few times on a synthetic volume (profiling target)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2510_20271_b200 as E
from paper_2510_20271_b200 import _lib

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
x = torch.empty((n, n, n), dtype=torch.float32, device="cuda")
_lib.check(_lib.lib().ecc_counter_grid(11, 0, x.numel(), _lib.ptr(x), _lib.stream_ptr(x)))
lo, hi, _ = E.device_minmax(x)
ts = E.thresholds_from_range(lo, hi, 1024)
for _ in range(reps):
    c = E.ecc_discrete(x, ts)
torch.cuda.synchronize()
print("ok", int(c[-1]))

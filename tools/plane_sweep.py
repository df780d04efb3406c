"""Device time of a slab sweep vs its single-plane boundary sweeps (the overlapped multi-GPU step)."""
import sys, torch
sys.path.insert(0, ".")
import paper_2510_20271_b200 as E
from paper_2510_20271_b200 import _lib, distributed as D
x = torch.empty((514, 512, 512), device="cuda")
_lib.check(_lib.lib().ecc_counter_grid(11, 0, x.numel(), _lib.ptr(x), _lib.stream_ptr(x)))
taus = E.thresholds_from_range(0.0, 1.0, 1024)
def t(fn, reps=50):
    for _ in range(5): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps
full = t(lambda: D._cuda_slab_hist(x, 1, 513, taus))
one = t(lambda: D._cuda_slab_hist(x, 1, 2, taus))
inner = t(lambda: D._cuda_slab_hist(x[1:-1], 1, 511, taus))
print(f"512 planes {full*1e3:.1f} us, one plane {one*1e3:.1f} us, interior 510 {inner*1e3:.1f} us, overlapped path {inner*1e3 + 2*one*1e3:.1f} us")

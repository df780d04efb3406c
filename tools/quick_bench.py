"""Quick device timings of the hot kernels (development aid, not the bench)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2510_20271_b200 as E

def timeit(fn, reps=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        s.record(); fn(); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
    return float(np.median(ts))

dev = torch.device("cuda")
for n in (512, 1024):
    x = torch.empty((n, n, n), dtype=torch.float32, device=dev)
    E._lib.check(E._lib.lib().ecc_counter_grid(11, 0, x.numel(), E._lib.ptr(x), E._lib.stream_ptr(x)))
    lo, hi, _ = E.device_minmax(x)
    ts = E.thresholds_from_range(lo, hi, 1024)
    ms = timeit(lambda: E.histogram_device(x, ts))
    print(f"hist {n}^3 f32 B=1024: {ms:.3f} ms  {x.numel()/ms/1e6:.1f} Gvox/s  {4*x.numel()/ms/1e6:.0f} GB/s", flush=True)
    ms = timeit(lambda: E.device_minmax(x))
    print(f"minmax {n}^3: {ms:.3f} ms", flush=True)
    del x
# soft C3-like: 8 images of 1024^2, B=256
N = 8
x = torch.rand((N, 1024, 1024), device=dev)
m = E.SoftECC(np.linspace(-0.4, 1.4, 256), [1.0, 2.0], alpha=0.3, lam=50.0).to(dev)
def step():
    chi = m(x)
    chi.sum().backward()
ms = timeit(step, reps=5)
pairs = x.numel() * 256
print(f"soft fwd+bwd {N}x1024^2 B=256: {ms:.2f} ms  {x.numel()/ms/1e6:.2f} Gvox/s  {pairs/ms/1e9:.2f} Tpairs/s(per pass x2)", flush=True)

"""Device time of histogram_device on the 512^3 / 1024^3 counter volumes (A/B of library builds via ECC_B200_LIB)."""
import sys, torch
sys.path.insert(0, ".")
import paper_2510_20271_b200 as E
from paper_2510_20271_b200 import _lib
for n in (512, 1024):
    x = torch.empty((n, n, n), device="cuda")
    _lib.check(_lib.lib().ecc_counter_grid(11, 0, x.numel(), _lib.ptr(x), _lib.stream_ptr(x)))
    ts = E.thresholds_from_range(0.0, 1.0, 1024)
    for _ in range(3): E.histogram_device(x, ts)
    torch.cuda.synchronize()
    best = 1e9
    for r in range(5):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(10): E.histogram_device(x, ts)
        e.record(); torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e) / 10)
    print(n, f"{best:.4f} ms")
    del x; torch.cuda.empty_cache()

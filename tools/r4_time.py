"""Back-to-back device time of the rank4 sweep at 512^3 and 1024^3 (1024 uniform
thresholds) for comparing compile-time library variants, e.g. the
ECC_R4_STRIP phase-cost builds (development aid).

    ECC_B200_LIB=tools/_v/<name>.so python tools/r4_time.py
"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2510_20271_b200 as E  # noqa: E402
from paper_2510_20271_b200 import _lib  # noqa: E402

L = _lib.lib()
ts = E.thresholds_from_range(0.0, 1.0, 1024)
res = []
for n in (512, 1024):
    x = torch.empty((n, n, n), device="cuda")
    _lib.check(L.ecc_counter_grid(11, 0, x.numel(), _lib.ptr(x), _lib.stream_ptr(x)))
    for _ in range(3):
        E.histogram_device(x, ts)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(10):
            E.histogram_device(x, ts)
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e) / 10)
    res.append(f"{n}^3 {best * 1e3:8.1f} us {n ** 3 / best / 1e6:6.1f} Gvox/s {4 * n ** 3 / best / 1e6 / 6535.1:.3f} of HBM")
    del x
    torch.cuda.empty_cache()
print(" | ".join(res))

"""C2 (512^3) device time under forced dynamic unit sizes (development aid)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2510_20271_b200 as E
from paper_2510_20271_b200 import _lib
n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
x = torch.empty((n, n, n), dtype=torch.float32, device="cuda")
_lib.check(_lib.lib().ecc_counter_grid(11, 0, x.numel(), _lib.ptr(x), _lib.stream_ptr(x)))
lo, hi, _ = E.device_minmax(x)
ts = E.thresholds_from_range(lo, hi, 1024)
table, binning = ts.device_table(_lib.DTYPE_F32, x.device)
hist = torch.empty(1025, dtype=torch.int64, device="cuda")
d = _lib.dims_arg(x.shape)
def run():
    _lib.check(_lib.lib().ecc_histogram(_lib.ptr(x), _lib.DTYPE_F32, 3, _lib.ptr(d), 1, _lib.ptr(table),
                                        _lib.ctypes.byref(binning), _lib.ptr(hist), _lib.stream_ptr(x)))
for rnd in range(2):
    for z in ([int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else [0, 4, 6, 8, 10, 12, 16, 24, 32]):
        with _lib.variant(zunit=z):
            for _ in range(3): run()
            torch.cuda.synchronize()
            best = 1e9
            for r in range(5):
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                for _ in range(10): run()
                e.record(); torch.cuda.synchronize()
                best = min(best, s.elapsed_time(e) / 10)
            if rnd == 1:
                print(f"zunit {z:3d}: {best:.4f} ms {n**3/best/1e6:.1f} Gvox/s", flush=True)

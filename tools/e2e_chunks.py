"""e2e timing of ecc_discrete_host for several chunk sizes (development aid)."""
import sys, time
import torch
sys.path.insert(0, ".")
import paper_2510_20271_b200 as E
from paper_2510_20271_b200 import _lib

P = 512
x = torch.empty((P, 512, 512), dtype=torch.float32, device="cuda")
_lib.check(_lib.lib().ecc_counter_grid(3, 0, x.numel(), _lib.ptr(x), _lib.stream_ptr(x)))
host = torch.empty(x.shape, dtype=torch.float32, pin_memory=True)
host.copy_(x.cpu())
lo, hi, _ = E.device_minmax(x)
ts = E.thresholds_from_range(lo, hi, 1024)
xdev = torch.empty_like(x)
def whole():
    xdev.copy_(host, non_blocking=True)
    return E.ecc_discrete(xdev, ts).cpu()
def timeit(fn, reps=8):
    fn(); fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) * 1e3 / reps
print(f"whole copy + kernel: {timeit(whole):.2f} ms")
ref = whole()
for res in (False, True):
    for cp in (16, 32, 64, 128, 256):
        assert torch.equal(E.ecc_discrete_host(host, ts, chunk_planes=cp, resident=res).cpu(), ref)
        ms = timeit(lambda: E.ecc_discrete_host(host, ts, chunk_planes=cp, resident=res).cpu())
        print(f"host streaming resident={res} chunk {cp}: {ms:.3f} ms")

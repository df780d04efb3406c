"""A/B of library builds (ECC_B200_LIB) on one volume: device time of the
histogram kernel, back-to-back launches between CUDA events; every build must
produce the same histogram (development aid)."""
import os, subprocess, sys, json
libs = sys.argv[1].split(",")
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
child = r'''
import sys, json, numpy as np, torch
sys.path.insert(0, ".")
import paper_2510_20271_b200 as E
from paper_2510_20271_b200 import _lib
n = int(sys.argv[1])
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
    return hist
h = run().cpu().numpy().reshape(-1)
for _ in range(3): run()
torch.cuda.synchronize()
best = 1e9
for r in range(5):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5): run()
    e.record(); torch.cuda.synchronize()
    best = min(best, s.elapsed_time(e) / 5)
print(json.dumps({"ms": best, "h": int(np.bitwise_xor.reduce(h.view(np.uint64)))}))
'''
res = {}
for rnd in range(2):
    for L in libs:
        env = dict(os.environ)
        if L and L != "default":
            env["ECC_B200_LIB"] = L if L.endswith(".so") else f"tools/_v/{L}.so"
        out = subprocess.run([sys.executable, "-c", child, str(n)], env=env, capture_output=True, text=True)
        try:
            d = json.loads(out.stdout.strip().splitlines()[-1])
        except Exception:
            print(L, "FAILED", out.stderr[-1500:]); continue
        res.setdefault(L, []).append(d)
hs = {d["h"] for v in res.values() for d in v}
print(f"{n}^3 histogram checksums agree: {len(hs) == 1}")
for L, v in res.items():
    ms = min(d["ms"] for d in v)
    print(f"{L:16s} {ms:.4f} ms {n**3/ms/1e6:7.1f} Gvox/s frac {4*n**3/ms/1e6/6535.1:.3f}", flush=True)

"""3D soft ECC forward+backward timing (C4-like, one GPU)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2510_20271_b200 as E

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
N = int(sys.argv[2]) if len(sys.argv) > 2 else 1
x = torch.rand((N, n, n, n), device="cuda")
v = np.array([1.0, 2.0, -0.5]); u = v / np.linalg.norm(v)
span = 0.3 * np.abs(u).sum()
m = E.SoftECC(np.linspace(-span, 1 + span, 257)[1:], v, alpha=0.3, lam=50.0).cuda()
def step():
    m.zero_grad(set_to_none=True)
    m(x).sum().backward()
step(); torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(3): step()
e.record(); torch.cuda.synchronize()
ms = s.elapsed_time(e) / 3
print(f"soft3d {N}x{n}^3 B=256: {ms:.2f} ms/step  {N*n**3/ms/1e6:.2f} Gvox/s")

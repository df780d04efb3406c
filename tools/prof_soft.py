"""Soft ECC forward+backward on a C3-like batch (profiling target)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2510_20271_b200 as E

N = int(sys.argv[1]) if len(sys.argv) > 1 else 8
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
x = torch.rand((N, 1024, 1024), device="cuda")
m = E.SoftECC(np.linspace(-0.67, 1.67, 256), [1.0, 2.0], alpha=0.3, lam=50.0).cuda()
for _ in range(reps):
    m.zero_grad()
    m(x).sum().backward()
torch.cuda.synchronize()
print("ok")

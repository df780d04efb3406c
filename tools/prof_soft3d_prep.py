"""Run the C4-sized soft module (1024^3, B = 256) once: profiling target for the
3-D prepare and the soft kernels."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2510_20271_b200 as E

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
v = np.array([1.0, 2.0, -0.5])
m = E.SoftECC(np.linspace(-0.5, 1.5, 256), v, alpha=0.3, lam=50.0).cuda()
x = torch.rand((1, n, n, n), device="cuda")
for _ in range(2):
    m(x).sum().backward()
torch.cuda.synchronize()
print("ok")

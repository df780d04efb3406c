"""C4 e2e (one 1024^3 item from pinned host memory through soft_step_host,
forward + backward, chi and gradients to the host) for several z-slab sizes;
slab = 1024 is the unstreamed order (development aid)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2510_20271_b200 as E  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
slabs = [int(a) for a in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["1024", "128", "64", "32"])]
B, v = 256, [1.0, 2.0, -0.5]
u = np.asarray(v) / np.linalg.norm(v)
span = 0.3 * np.abs(u).sum()
taus = np.linspace(-span, 1.0 + span, B + 1)[1:]
m = E.SoftECC(taus, v, alpha=0.3, lam=50.0).cuda()
host = torch.empty((1, n, n, n), dtype=torch.float32, pin_memory=True)
host.uniform_()
up = torch.ones((1, B), dtype=torch.float64, device="cuda")
for slab in slabs:
    def step():
        m.zero_grad(set_to_none=True)
        chi = E.soft_step_host(m, host, up, micro=1, slab_planes=slab)
        return chi.cpu(), m.taus.grad.cpu(), m.v.grad.cpu(), m.alpha.grad.cpu()
    ref = step()
    torch.cuda.synchronize()
    ts = []
    for _ in range(6):
        t0 = time.perf_counter()
        out = step()
        ts.append((time.perf_counter() - t0) * 1e3)
    same = all(torch.equal(a, b) for a, b in zip(ref, out))
    print(f"slab {slab:5d}: {min(ts):8.1f} ms/step (median {np.median(ts):.1f})  repeatable: {same}", flush=True)

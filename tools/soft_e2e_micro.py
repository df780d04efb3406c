"""C3 soft e2e (soft_step_host) wall time per step for several micro-batch sizes (development aid)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2510_20271_b200 as E

N, H, W, B = 128, 1024, 1024, 256
v = np.array([1.0, 2.0]); u = v / np.linalg.norm(v); span = 0.3 * np.abs(u).sum()
taus = np.linspace(-span, 1.0 + span, B + 1)[1:]
m = E.SoftECC(taus, v, alpha=0.3, lam=50.0).cuda()
host = torch.rand((N, H, W)).pin_memory()
up = torch.ones((N, B), dtype=torch.float64, device="cuda")
for micro in [int(a) for a in (sys.argv[1].split(",") if len(sys.argv) > 1 else "8,16,32")]:
    def step():
        m.zero_grad(set_to_none=True)
        chi = E.soft_step_host(m, host, up, micro=micro)
        return chi.cpu(), m.taus.grad.cpu()
    step(); torch.cuda.synchronize()
    best = 1e9
    for _ in range(3):
        t0 = time.perf_counter()
        for _ in range(3):
            step()
        torch.cuda.synchronize()
        best = min(best, (time.perf_counter() - t0) / 3 * 1e3)
    print(f"micro {micro:3d}: {best:.2f} ms/step", flush=True)

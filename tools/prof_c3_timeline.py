"""Kernel timeline of the C3 soft step (torch.profiler / CUPTI, no ncu): per-kernel device time and the
idle time between kernels within a step (development aid)."""
import sys
import numpy as np
import torch
from torch.profiler import profile, ProfilerActivity
sys.path.insert(0, ".")
import paper_2510_20271_b200 as E

N, H, W, B = 128, 1024, 1024, 256
v = np.array([1.0, 2.0]); u = v / np.linalg.norm(v); span = 0.3 * np.abs(u).sum()
taus = np.linspace(-span, 1.0 + span, B + 1)[1:]
m = E.SoftECC(taus, v, alpha=0.3, lam=50.0).cuda()
x = torch.rand((N, H, W), device="cuda")
up = torch.ones((N, B), dtype=torch.float64, device="cuda")
def step():
    m.zero_grad(set_to_none=True)
    m(x).backward(up)
for _ in range(3):
    step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        step()
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
ev.sort(key=lambda e: e.time_range.start)
tot = {}
for e in ev:
    tot.setdefault(e.name[:60], [0.0, 0])
    tot[e.name[:60]][0] += e.time_range.elapsed_us()
    tot[e.name[:60]][1] += 1
span_us = ev[-1].time_range.end - ev[0].time_range.start
busy = sum(e.time_range.elapsed_us() for e in ev)
print(f"3 steps: span {span_us/3:.0f} us/step, kernels {busy/3:.0f} us/step, gaps {(span_us - busy)/3:.0f} us/step")
for k, (t, c) in sorted(tot.items(), key=lambda kv: -kv[1][0])[:15]:
    print(f"{t/3:9.1f} us/step  {c//3:3d}x  {k}")

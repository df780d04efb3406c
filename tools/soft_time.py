"""Device time of the SoftECC module's forward and backward on C3-shaped images
(128 x 1024^2, B = 256) and a 256 x 512^2 3-D item, for comparing compile-time
library variants (ECC_B200_LIB=tools/_v/<name>.so), plus a digest of the outputs
(development aid).

    ECC_B200_LIB=tools/_v/a.so python tools/soft_time.py [out.npz]
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2510_20271_b200 as E  # noqa: E402


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    return float(np.median(ts))


out = {}
for name, shape, v in (("c3", (128, 1024, 1024), [1.0, 2.0]), ("c4s", (1, 256, 512, 512), [1.0, 2.0, -0.5])):
    B, lam, alpha = 256, 50.0, 0.3
    u = np.asarray(v) / np.linalg.norm(v)
    span = alpha * np.abs(u).sum()
    taus = np.linspace(-span, 1.0 + span, B + 1)[1:]
    g = torch.Generator(device="cuda").manual_seed(5)
    x = torch.rand(shape, device="cuda", generator=g).requires_grad_(True)
    up = torch.rand((shape[0], B), device="cuda", dtype=torch.float64, generator=g) + 0.5
    m = E.SoftECC(taus, v, alpha=alpha, lam=lam).cuda()
    state = {}

    def fwd():
        state["chi"] = m(x)

    def bwd():
        x.grad = None
        m.zero_grad()
        state["chi"].backward(up, retain_graph=True)

    tf = timed(fwd)
    fwd()
    tb = timed(bwd)
    tt = timed(lambda: (fwd(), bwd()))
    chi = state["chi"].detach().cpu().numpy()
    gx = x.grad.cpu().numpy()
    print(f"{name}: forward {tf:.3f} ms  backward {tb:.3f} ms  step {tt:.3f} ms  "
          f"chi sum {chi.sum():.9e}  dx norm {np.linalg.norm(gx):.9e}", flush=True)
    out[name + "_chi"] = chi
    out[name + "_dx"] = gx[:2] if gx.ndim == 3 else gx[0, :8]
    out[name + "_taus"] = m.taus.grad.cpu().numpy() if m.taus.grad is not None else np.zeros(1)
    del x, m, state
    torch.cuda.empty_cache()
if len(sys.argv) > 1:
    np.savez(sys.argv[1], **out)

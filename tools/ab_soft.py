"""A/B of the soft kernels (ecc_set_variant soft_band / soft_g ...): device time of the
SoftECC module's forward and backward on C3-shaped images and a C4-shaped
volume, and the normwise distance of every output between the variants
(development aid)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2510_20271_b200 as E  # noqa: E402
from paper_2510_20271_b200 import _lib  # noqa: E402


def case(shape, v):
    B, lam, alpha = 256, 50.0, 0.3
    u = np.asarray(v) / np.linalg.norm(v)
    span = alpha * np.abs(u).sum()
    taus = np.linspace(-span, 1.0 + span, B + 1)[1:]
    g = torch.Generator(device="cuda").manual_seed(5)
    x = torch.rand(shape, device="cuda", generator=g)
    up = torch.rand((shape[0], B), device="cuda", dtype=torch.float64, generator=g) + 0.5
    return E.SoftECC(taus, v, alpha=alpha, lam=lam).cuda(), x, up


def run(m, x, up, reps):
    xs = x.clone().requires_grad_(True)
    m.zero_grad()
    chi = m(xs)
    (chi * up).sum().backward()
    outs = [chi.detach().clone(), xs.grad.clone(), m.taus.grad.clone(), m.v.grad.clone(), m.alpha.grad.clone()]
    tf, tb = [], []
    for _ in range(reps):
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        xs.grad = None
        e0.record()
        chi = m(xs)
        e1.record()
        (chi * up).sum().backward()
        e2.record()
        torch.cuda.synchronize()
        tf.append(e0.elapsed_time(e1))
        tb.append(e1.elapsed_time(e2))
    return outs, float(np.median(tf)), float(np.median(tb))


def nw(a, b):
    a, b = a.double().cpu().numpy().ravel(), b.double().cpu().numpy().ravel()
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


cases = {"c3": ((16, 1024, 1024), [1.0, 2.0]), "c3b": ((128, 1024, 1024), [1.0, 2.0]),
         "c4": ((1, 512, 512, 512), [1.0, 2.0, -0.5])}
sel = sys.argv[1].split(",") if len(sys.argv) > 1 else ["c3", "c4"]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
# variants: "soft_band=0:soft_g=1" ...; the first is the reference of the distances
vars_ = sys.argv[3].split(",") if len(sys.argv) > 3 else ["soft_band=0", "soft_band=1"]
for name in sel:
    shape, v = cases[name]
    m, x, up = case(shape, v)
    res = {}
    for rnd in range(2):
        for var in vars_:
            kw = dict(kv.split("=") for kv in var.split(":"))
            with _lib.variant(**kw):
                outs, tf, tb = run(m, x, up, reps)
            r = res.setdefault(var, [outs, [], []])
            r[1].append(tf)
            r[2].append(tb)
    ref = res[vars_[0]][0]
    for var in vars_:
        d = [nw(a, b) for a, b in zip(res[var][0], ref)]
        print(f"{name} {var:24s} fwd {min(res[var][1]):8.3f} ms  bwd {min(res[var][2]):8.3f} ms   "
              f"vs first: chi {d[0]:.1e} dX {d[1]:.1e} dtau {d[2]:.1e} dv {d[3]:.1e} dalpha {d[4]:.1e}", flush=True)
    del m, x, up
    torch.cuda.empty_cache()

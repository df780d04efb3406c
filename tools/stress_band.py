"""Randomised band-vs-full check of the soft module (development aid): random shapes (2-D / 3-D, odd
sizes), random sorted non-uniform thresholds, lambda around the band condition, several G; the band
kernels must match the full ones (chi, dX, dtau normwise <= 1e-5; dv, dalpha <= 1e-4)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2510_20271_b200 as E
from paper_2510_20271_b200 import _lib
from paper_2510_20271_b200.soft import band_window

def nw(a, b):
    a, b = np.asarray(a, np.float64).ravel(), np.asarray(b, np.float64).ravel()
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))

def outs(m, x, up):
    xs = x.clone().requires_grad_(True)
    m.zero_grad()
    chi = m(xs)
    (chi * up).sum().backward()
    return [chi.detach().cpu().numpy(), xs.grad.cpu().numpy(), m.taus.grad.cpu().numpy(), m.v.grad.cpu().numpy(),
            m.alpha.grad.cpu().numpy()]

rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
ncase = int(sys.argv[2]) if len(sys.argv) > 2 else 40
bad = 0
nband = 0
for k in range(ncase):
    nd = int(rng.integers(2, 4))
    shape = (int(rng.integers(1, 4)),) + tuple(int(rng.integers(5, 90 if nd == 2 else 40)) for _ in range(nd))
    B = int(rng.integers(150, 369))
    v = rng.normal(size=nd)
    alpha = float(rng.uniform(0.0, 0.5))
    u = v / np.linalg.norm(v)
    span = alpha * np.abs(u).sum()
    taus = np.sort(rng.uniform(-span - 0.1, 1.0 + span + 0.1, B))
    lam = float(rng.uniform(10.0, 120.0))
    win = band_window(taus, lam)
    nband += win < B
    m = E.SoftECC(taus, v, alpha=alpha, lam=lam).cuda()
    x = torch.from_numpy(rng.random(shape).astype(np.float32)).cuda()
    up = torch.from_numpy(rng.uniform(0.5, 1.5, (shape[0], B))).cuda()
    g = int(rng.choice([0, 1, 2, 5]))
    with _lib.variant(soft_band=0, soft_g=g):
        full = outs(m, x, up)
    with _lib.variant(soft_g=g):
        band = outs(m, x, up)
    d = [nw(a, b) for a, b in zip(band, full)]
    ok = d[0] <= 1e-5 and d[1] <= 1e-5 and d[2] <= 1e-5 and d[3] <= 1e-4 and abs(float(band[4]) - float(full[4])) <= 1e-4 * max(abs(float(full[4])), 1e-3)
    if not ok:
        bad += 1
        print("MISMATCH", k, shape, B, round(lam, 2), win, g, ["%.1e" % t for t in d], flush=True)
print(f"{ncase} cases, {nband} in band mode, {bad} mismatches")

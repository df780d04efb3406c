"""Randomised row-word prepare vs the generic sweep (development aid): random 2-D / 3-D shapes, float32 /
float64, ties, alpha (incl. 0), occasional non-finite values; coefficients and centred field bit-exact."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2510_20271_b200 as E

rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
ncase = int(sys.argv[2]) if len(sys.argv) > 2 else 40
bad = 0
for k in range(ncase):
    nd = int(rng.integers(2, 4))
    dims = tuple(int(rng.integers(1, 120 if nd == 2 else 50)) for _ in range(nd))
    batch = int(rng.integers(1, 4))
    dtype = np.float32 if rng.random() < 0.7 else np.float64
    x = rng.random((batch,) + dims).astype(dtype)
    if rng.random() < 0.5:
        x = (np.round(x * 8) / 8).astype(dtype)          # ties
    if rng.random() < 0.15:
        idx = tuple(int(rng.integers(0, s)) for s in x.shape)
        x[idx] = rng.choice([np.nan, np.inf, -np.inf])
    alpha = 0.0 if rng.random() < 0.2 else float(rng.uniform(0.0, 0.5))
    u = E.reparametrize_direction(rng.normal(size=nd))
    p = E.soft._params(50.0, alpha, u, -0.5, 1.5, nd, 0.01)
    t = torch.from_numpy(x).cuda()
    c1, (f1, _) = E.soft.soft_prepare_device(t, dims, batch, p)
    with E._lib.variant(generic=1):
        c2, (f2, _) = E.soft.soft_prepare_device(t, dims, batch, p)
    if not (torch.equal(c1, c2) and torch.equal(f1.view(torch.int32), f2.view(torch.int32))):
        bad += 1
        print("MISMATCH", k, dims, batch, dtype.__name__, alpha, flush=True)
print(f"{ncase} cases, {bad} mismatches")

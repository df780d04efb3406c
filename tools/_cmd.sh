timeout 900 python -m pytest tests/test_gpu_discrete.py -m gpu -x -q --timeout 600 2>&1 | tail -3
python - <<'PY'
import torch, sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_2510_20271_b200 as E
for n in (512, 1024):
    x = torch.randint(0, 256, (n, n, n), dtype=torch.uint8, device="cuda")
    ts = E.ThresholdSet(np.arange(0.0, 256.0, 1.0))
    for _ in range(3): E.histogram_device(x, ts)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5): E.histogram_device(x, ts)
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 5
    print(f"u8 {n}^3 256 bins: {ms:.3f} ms {x.numel()/ms/1e6:.1f} Gvox/s")
PY

"""uint8 3D discrete ECC timing (development aid)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2510_20271_b200 as E

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
g = torch.Generator(device="cuda"); g.manual_seed(3)
x = torch.randint(0, 256, (n, n, n), dtype=torch.uint8, device="cuda", generator=g)
ts = E.ThresholdSet(list(range(256)))
for _ in range(3):
    E.histogram_device(x, ts)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(5):
    E.histogram_device(x, ts)
e.record(); torch.cuda.synchronize()
ms = s.elapsed_time(e) / 5
print(f"u8 {n}^3 B=256: {ms:.3f} ms  {x.numel() / ms / 1e6:.1f} Gvox/s")

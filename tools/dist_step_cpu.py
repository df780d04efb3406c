"""Host enqueue time vs wall time of one distributed C2 step (slab_histogram) under torchrun (development
aid: the multi-GPU step must not be CPU-bound; N = 1 measured 0.080 ms enqueue vs 0.241 ms per step)."""
import os, sys, time
sys.path.insert(0, ".")
import torch, torch.distributed as dist
import numpy as np
import paper_2510_20271_b200 as E
from paper_2510_20271_b200 import _lib, distributed as D
dev = torch.device("cuda", 0); torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=dev)
P, H, W = 512, 512, 512
padded = D.alloc_padded_slab(P, (H, W), torch.float32, dev)
own = padded[1:-1]
_lib.check(_lib.lib().ecc_counter_grid(11, 0, own.numel(), _lib.ptr(own), _lib.stream_ptr(own)))
taus = E.thresholds_from_range(0.0, 1.0, 1024)
for name, fn in [("slab_histogram", lambda: D.slab_histogram(padded, taus, depth=P)),
                 ("sweep only", lambda: D._cuda_slab_hist(own, 0, P, taus))]:
    for _ in range(5): fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(50): fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{name}: host enqueue {1e3*(t1-t0)/50:.3f} ms/step, wall {1e3*(t2-t0)/50:.3f} ms/step")
dist.destroy_process_group()

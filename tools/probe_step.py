"""Split the headline bench step (cfg 2 fused solve) into device kernels and host
gaps with the CUDA profiler API (torch.profiler / CUPTI); development probe."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_18413_b200 as cs  # noqa: E402

m = cs.model_logp_grad_hvp(cs.rosenbrock(a=0.0, b=0.1, scale1=1.0, scale2=1.0))
k = cs.HmcKernel(m, 0.5, 8, seed=0, T=100_000, dtype=torch.float32)
cfg = cs.DeerConfig(mode="diag-stochastic", clip=1.0)
s0 = torch.zeros(2, dtype=torch.float32, device="cuda")
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
for _ in range(5):
    cs.run_deer(k, s0, cfg)
torch.cuda.synchronize()
for fl in (False, True):
    ev, walls = [], []
    for _ in range(30):
        if fl:
            flush.fill_(1.0)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        a.record()
        cs.run_deer(k, s0, cfg)
        b.record()
        torch.cuda.synchronize()
        walls.append(time.perf_counter() - t0)
        ev.append(a.elapsed_time(b))
    print(f"flush={fl}: events {np.median(ev):.3f} ms (min {np.min(ev):.3f}), wall {1e3 * np.median(walls):.3f} ms")
from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    for _ in range(10):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        cs.run_deer(k, s0, cfg)
        torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=12))

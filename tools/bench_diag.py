"""Per-step timing of the headline solve under the bench's timing loop
(development): with / without the L2 flush and the NVML poller child."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2508_18413_b200 as cs  # noqa: E402

dev = torch.device("cuda", 0)
m = cs.model_logp_grad_hvp(cs.rosenbrock(a=0.0, b=0.1, scale1=1.0, scale2=1.0))
k = cs.HmcKernel(m, 0.5, 8, seed=0, T=100_000, dtype=torch.float32)
cfg = cs.DeerConfig(mode="diag-stochastic", clip=1.0)
s0 = torch.zeros(2, dtype=torch.float32, device=dev)
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
for _ in range(5):
    r = cs.run_deer(k, s0, cfg)
torch.cuda.synchronize()


def loop(tag, do_flush, n=20):
    ev, walls, dms = [], [], []
    for _ in range(n):
        if do_flush:
            flush.fill_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        a.record()
        r = cs.run_deer(k, s0, cfg)
        b.record()
        walls.append(time.perf_counter() - t0)
        dms.append(r.stats["device_ms"])
        ev.append((a, b))
    torch.cuda.synchronize()
    ms = [a.elapsed_time(b) for a, b in ev]
    print(f"{tag:28s} event ms p50 {np.median(ms):.3f} max {np.max(ms):.3f} | wall ms p50 {1e3*np.median(walls):.3f} "
          f"| kernel ms p50 {np.median(dms):.3f}  all={np.round(ms, 3).tolist()}")


loop("no flush", False)
loop("flush", True)
with bench.ClockSampler(0):
    loop("flush + poller", True)
    loop("no flush + poller", False)
loop("flush again", True)

"""Where the headline solve's host time goes (development)."""
import os
import sys
import time
import cProfile
import pstats

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_18413_b200 as cs  # noqa: E402

m = cs.model_logp_grad_hvp(cs.rosenbrock(a=0.0, b=0.1, scale1=1.0, scale2=1.0))
k = cs.HmcKernel(m, 0.5, 8, seed=0, T=100_000, dtype=torch.float32)
cfg = cs.DeerConfig(mode="diag-stochastic", clip=1.0)
s0 = torch.zeros(2, dtype=torch.float32, device="cuda")
for _ in range(10):
    cs.run_deer(k, s0, cfg)
torch.cuda.synchronize()


def t(fn, n=200):
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    return (time.perf_counter() - t0) / n * 1e6


print(f"desc()            {t(k.desc):7.1f} us")
print(f"torch.empty x2    {t(lambda: (torch.empty((100000, 2), device='cuda'), torch.empty(100000, dtype=torch.int32, device='cuda'))):7.1f} us")
walls, ker = [], []
for _ in range(50):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = cs.run_deer(k, s0, cfg)
    walls.append(time.perf_counter() - t0)
    ker.append(r.stats["device_ms"])
print(f"run_deer wall {1e3 * np.median(walls):.3f} ms, kernel {np.median(ker):.3f} ms")
pr = cProfile.Profile()
pr.enable()
for _ in range(200):
    cs.run_deer(k, s0, cfg)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)

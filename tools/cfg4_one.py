"""BASELINE cfg 4 (leapfrog, dense Gaussian D = 1000, L = 100, block2x2, f64):
solves for ncu / timing (dev probe): python tools/cfg4_one.py [n_solves]."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_18413_b200 as cs  # noqa: E402
from bench_configs import cfg4_chol  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 3
D, eps, L = 1000, 0.05, 100
m = cs.model_logp_grad_hvp(cs.gaussian(np.zeros(D), cfg4_chol(D)))
x0 = np.random.default_rng(1).normal(size=D)
v0 = np.random.default_rng(2).normal(size=D)
s0 = np.concatenate([x0, v0 + 0.5 * eps * m.grad(torch.as_tensor(x0, device="cuda")).cpu().numpy()])
lf = cs.LeapfrogSystem(m, eps, L, dtype=torch.float64)
cfg = cs.DeerConfig(mode="block2x2-stochastic")
for _ in range(n):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = cs.run_deer(lf, s0, cfg)
    torch.cuda.synchronize()
    print(f"{1e3 * (time.perf_counter() - t0):.3f} ms, {r.iterations} iterations", flush=True)

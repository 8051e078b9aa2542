"""Split the headline solve's wall time into host work and device time (dev probe)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_18413_b200 as cs  # noqa: E402
from paper_2508_18413_b200 import deer  # noqa: E402

m = cs.model_logp_grad_hvp(cs.rosenbrock(a=0.0, b=0.1, scale1=1.0, scale2=1.0))
k = cs.HmcKernel(m, 0.5, 8, seed=0, T=100_000, dtype=torch.float32)
cfg = cs.DeerConfig(mode="diag-stochastic", clip=1.0)
s0 = torch.zeros(2, dtype=torch.float32, device="cuda")
for _ in range(5):
    cs.run_deer(k, s0, cfg)
torch.cuda.synchronize()
lib = cs._lib.load()
orig = lib.cs_deer_solve
tt = []


def timed_solve(*a):
    t0 = time.perf_counter()
    r = orig(*a)
    tt.append(time.perf_counter() - t0)
    return r


class Wrap:
    def __getattr__(self, n):
        return timed_solve if n == "cs_deer_solve" else getattr(lib, n)


deer._lib.load = lambda: Wrap()
walls = []
for _ in range(30):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    cs.run_deer(k, s0, cfg)
    torch.cuda.synchronize()
    walls.append(time.perf_counter() - t0)
print(f"run_deer wall {1e3 * np.median(walls):.3f} ms, inside cs_deer_solve {1e3 * np.median(tt):.3f} ms "
      f"-> python-side {1e3 * (np.median(walls) - np.median(tt)):.3f} ms")

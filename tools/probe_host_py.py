"""cProfile of run_deer's Python side on the headline solve (development probe)."""
import cProfile
import os
import pstats
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_18413_b200 as cs  # noqa: E402

m = cs.model_logp_grad_hvp(cs.rosenbrock(a=0.0, b=0.1, scale1=1.0, scale2=1.0))
k = cs.HmcKernel(m, 0.5, 8, seed=0, T=100_000, dtype=torch.float32)
cfg = cs.DeerConfig(mode="diag-stochastic", clip=1.0)
s0 = torch.zeros(2, dtype=torch.float32, device="cuda")
for _ in range(5):
    cs.run_deer(k, s0, cfg)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(200):
    cs.run_deer(k, s0, cfg)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)

import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2508_18413_b200 as cs
k = cs.GibbsKernel(cs.generate_eight_schools(), seed=0, T=1_000_000, dtype=torch.float32)
cfg = cs.DeerConfig(mode="diag-stochastic", hutchinson_samples=3, preconditioner=k.recommended_preconditioner(), max_iters=int(sys.argv[1]) if len(sys.argv) > 1 else 400)
r = cs.run_deer(k, k.initial_state(), cfg)
print(r.iterations, r.converged)

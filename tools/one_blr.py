"""One short cfg3 BLR MALA diag solve (profiling target)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_18413_b200 as cs  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 20_000
dt = torch.float64 if (len(sys.argv) > 2 and sys.argv[2] == "f64") else torch.float32
X, y, _ = cs.synthetic_credit_like(seed=20250819, n=1000, dim=100)
m = cs.model_logp_grad_hvp(cs.blr(X, y, 1.0))
k = cs.MalaKernel(m, 0.003, seed=4, T=T, dtype=dt)
r = cs.run_deer(k, np.zeros(100), cs.DeerConfig(mode="diag-stochastic", max_iters=3))
torch.cuda.synchronize()
print("iters", r.iterations, r.stats)

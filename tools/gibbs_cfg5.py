"""BASELINE cfg 5 (Gibbs eight schools, T = 1M, diag x3 + preconditioner): one
solve for ncu (argv[1] = max_iters), or timed solves with --time (dev probe)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_18413_b200 as cs  # noqa: E402

k = cs.GibbsKernel(cs.generate_eight_schools(), seed=0, T=1_000_000, dtype=torch.float32)
mi = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 400
cfg = cs.DeerConfig(mode="diag-stochastic", hutchinson_samples=3, preconditioner=k.recommended_preconditioner(),
                    max_iters=mi)
s0 = k.initial_state()
r = cs.run_deer(k, s0, cfg)
if "--time" in sys.argv:
    ts = []
    for _ in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = cs.run_deer(k, s0, cfg)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    ts.sort()
    print(f"cfg5 T=1M: {1e3 * ts[2]:.1f} ms (median of 5), {r.iterations} iterations, converged={r.converged}")
else:
    print(r.iterations, r.converged)

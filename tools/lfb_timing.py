"""Outer run_deer over an HMC chain in parallel-leapfrog mode: batched inner solves vs the per-row loop."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_18413_b200 as cs  # noqa: E402
from paper_2508_18413_b200.samplers import hmc_chain_system  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
m = cs.model_logp_grad_hvp(cs.rosenbrock(b=0.1, scale2=1.0))
for eng in ("auto", "host"):
    k = hmc_chain_system(m, eps=0.2, L=16, seed=5, T=T, leapfrog_mode="parallel",
                         leapfrog_cfg=cs.DeerConfig(mode="block2x2-stochastic", engine=eng))
    torch.cuda.synchronize(); t0 = time.perf_counter()
    r = cs.run_deer(k, np.array([0.5, -0.5]), cs.DeerConfig(mode="diag-stochastic", clip=1.0, max_iters=60))
    torch.cuda.synchronize()
    print(f"inner={eng}: T={T} outer iterations={r.iterations} converged={r.converged} "
          f"{time.perf_counter() - t0:.2f} s, fallbacks={k.n_leapfrog_fallbacks}", flush=True)

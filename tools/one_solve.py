"""Run exactly one solve of a BASELINE config (for launch lists under ncu)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_18413_b200 as cs  # noqa: E402
from tools.bench_configs import cfg4_chol  # noqa: E402


def main():
    which = sys.argv[1]
    if which == "2":  # the bench's headline solve, several times (profile the 4th launch)
        m = cs.model_logp_grad_hvp(cs.rosenbrock(a=0.0, b=0.1, scale1=1.0, scale2=1.0))
        k = cs.HmcKernel(m, 0.5, 8, seed=0, T=100_000, dtype=torch.float32)
        for _ in range(5):
            r = cs.run_deer(k, np.zeros(2), cs.DeerConfig(mode="diag-stochastic", clip=1.0))
    elif which == "4":
        D, eps, L = 1000, 0.05, 100
        m = cs.model_logp_grad_hvp(cs.gaussian(np.zeros(D), cfg4_chol(D)))
        x0 = np.random.default_rng(1).normal(size=D)
        v0 = np.random.default_rng(2).normal(size=D)
        s0 = np.concatenate([x0, v0 + 0.5 * eps * m.grad(torch.as_tensor(x0, device="cuda")).cpu().numpy()])
        lf = cs.LeapfrogSystem(m, eps, L, dtype=torch.float64)
        r = cs.run_deer(lf, s0, cs.DeerConfig(mode="block2x2-stochastic"))
    elif which == "5":
        k = cs.GibbsKernel(cs.generate_eight_schools(), seed=0, T=int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000,
                           dtype=torch.float32)
        s0 = k.initial_state()
        cfg = cs.DeerConfig(mode="diag-stochastic", hutchinson_samples=3, preconditioner=k.recommended_preconditioner(),
                            max_iters=400)
        r = cs.run_deer(k, s0, cfg)
    elif which == "3d":  # cfg3 "full": dense Newton, f32 states (the tcgen05 Hessian path)
        X, y, _ = cs.synthetic_credit_like(seed=20250819, n=1000, dim=100)
        m = cs.model_logp_grad_hvp(cs.blr(X, y, 1.0))
        k = cs.MalaKernel(m, 0.003, seed=4, T=100_000, dtype=torch.float32)
        r = cs.run_deer(k, np.zeros(100), cs.DeerConfig(mode="dense", max_iters=int(sys.argv[2]) if len(sys.argv) > 2 else None))
    elif which == "3":
        X, y, _ = cs.synthetic_credit_like(seed=20250819, n=1000, dim=100)
        m = cs.model_logp_grad_hvp(cs.blr(X, y, 1.0))
        k = cs.MalaKernel(m, 0.003, seed=4, T=100_000, dtype=torch.float64)
        r = cs.run_deer(k, np.zeros(100), cs.DeerConfig(mode="diag-stochastic", max_iters=int(sys.argv[2]) if len(sys.argv) > 2 else None))
    torch.cuda.synchronize()
    print("iterations", r.iterations, "converged", r.converged)


if __name__ == "__main__":
    main()

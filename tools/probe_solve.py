"""Time whole-chain solves for the BASELINE configs (development probe)."""
import argparse
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_18413_b200 as cs  # noqa: E402


def make(cfg, T, dtype):
    if cfg == "hmc":
        m = cs.model_logp_grad_hvp(cs.rosenbrock(a=0.0, b=0.1, scale1=1.0, scale2=1.0))
        return cs.HmcKernel(m, 0.5, 8, seed=0, T=T, dtype=dtype), np.zeros(2), cs.DeerConfig(mode="diag-stochastic", clip=1.0)
    if cfg == "mala":
        m = cs.model_logp_grad_hvp(cs.gaussian([1.0, -1.0], [[1.0, 0.0], [-0.6, 1.2]]))
        return cs.MalaKernel(m, 0.4, seed=0, T=T, dtype=dtype), np.zeros(2), cs.DeerConfig(mode="dense")
    if cfg == "gibbs":
        k = cs.GibbsKernel(cs.generate_eight_schools(), seed=0, T=T, dtype=dtype)
        return k, k.initial_state(), cs.DeerConfig(mode="diag-stochastic", hutchinson_samples=3,
                                                   preconditioner=k.recommended_preconditioner(), max_iters=400)
    raise KeyError(cfg)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", default="hmc")
    ap.add_argument("--T", type=int, nargs="+", default=[100_000])
    ap.add_argument("--dtype", default="f32")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--engine", default="auto")
    a = ap.parse_args()
    dtype = torch.float32 if a.dtype == "f32" else torch.float64
    for T in a.T:
        k, s0, cfg = make(a.cfg, T, dtype)
        cfg.engine = a.engine
        r = cs.run_deer(k, s0, cfg)
        torch.cuda.synchronize()
        ts = []
        for _ in range(a.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            r = cs.run_deer(k, s0, cfg)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = float(np.median(ts))
        print(f"{a.cfg} T={T} {a.dtype} iters={r.iterations} conv={r.converged} ms={ms:.3f} "
              f"per-iter={1e3 * ms / max(1, r.iterations + 1):.1f}us samples/s={T / ms * 1e3:.3e} stats={r.stats}",
              flush=True)


if __name__ == "__main__":
    main()

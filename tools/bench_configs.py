"""Time every BASELINE.json config on one B200 (development table for DESIGN.md).

Each row: one full run_deer solve from device-resident noise (median of reps),
Newton iterations, converged samples/s; the CPU numbers are the reference's own
timings from BASELINE.md section 3 (8-vCPU host, numba), quoted for context.
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_18413_b200 as cs  # noqa: E402


def timed(fn, reps):
    if reps == 0:  # one cold run, timed (long solves are their own warm-up)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        r = fn()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b), r
    r = fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        r = fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts)), r


def cfg4_chol(D=1000):
    rng = np.random.default_rng(0)
    Q, _ = np.linalg.qr(rng.normal(size=(D, D)))
    lam = np.exp(rng.uniform(np.log(0.1), np.log(10.0), D))
    return np.linalg.cholesky((Q * lam) @ Q.T)


def main():
    which = sys.argv[1:] or ["1", "1r", "2", "3", "4", "5"]
    dt = torch.float32
    rows = []
    if "1" in which:
        m = cs.model_logp_grad_hvp(cs.gaussian([1.0, -1.0], [[1.0, 0.0], [-0.6, 1.2]]))
        k = cs.MalaKernel(m, 0.4, seed=0, T=10_000, dtype=dt)
        ms, r = timed(lambda: cs.run_deer(k, np.zeros(2), cs.DeerConfig(mode="dense")), 20)
        rows.append(("cfg1 MALA Gaussian 2D T=10K dense", ms, r, 10_000, 52_400))
    if "1r" in which:
        m = cs.model_logp_grad_hvp(cs.rosenbrock(b=0.1, scale2=1.0))
        k = cs.MalaKernel(m, 0.5, seed=0, T=10_000, dtype=dt)
        ms, r = timed(lambda: cs.run_deer(k, np.zeros(2), cs.DeerConfig(mode="dense")), 20)
        rows.append(("cfg1' MALA Rosenbrock 2D T=10K dense", ms, r, 10_000, 50_000))
    if "2" in which:
        m = cs.model_logp_grad_hvp(cs.rosenbrock(a=0.0, b=0.1, scale1=1.0, scale2=1.0))
        k = cs.HmcKernel(m, 0.5, 8, seed=0, T=100_000, dtype=dt)
        ms, r = timed(lambda: cs.run_deer(k, np.zeros(2), cs.DeerConfig(mode="diag-stochastic", clip=1.0)), 20)
        rows.append(("cfg2 HMC Rosenbrock T=100K diag+clip", ms, r, 100_000, 34_500))
    if "3" in which:
        X, y, _ = cs.synthetic_credit_like(seed=20250819, n=1000, dim=100)
        m = cs.model_logp_grad_hvp(cs.blr(X, y, 1.0))
        k = cs.MalaKernel(m, 0.003, seed=4, T=100_000, dtype=torch.float64)
        ms, r = timed(lambda: cs.run_deer(k, np.zeros(100), cs.DeerConfig(mode="diag-stochastic")), 1)
        rows.append(("cfg3 MALA BLR D=100 T=100K diag (f64)", ms, r, 100_000, None))
    for key, T3 in (("3d10k", 10_000), ("3d", 100_000)):
        if key not in which:
            continue
        # cfg3 "full": dense Newton (Jacobians from the system's jvps, wide dense scan)
        X, y, _ = cs.synthetic_credit_like(seed=20250819, n=1000, dim=100)
        m = cs.model_logp_grad_hvp(cs.blr(X, y, 1.0))
        k = cs.MalaKernel(m, 0.003, seed=4, T=T3, dtype=dt)
        t0 = time.perf_counter()
        ms, r = timed(lambda: cs.run_deer(k, np.zeros(100), cs.DeerConfig(mode="dense")), 0)
        print(f"  cfg3 dense T={T3}: {time.perf_counter() - t0:.1f} s incl. warm-up", flush=True)
        rows.append((f"cfg3 MALA BLR D=100 T={T3} dense (f32)", ms, r, T3, None))
    if "4" in which:
        D, eps, L = 1000, 0.05, 100
        Lc = cfg4_chol(D)
        m = cs.model_logp_grad_hvp(cs.gaussian(np.zeros(D), Lc))
        x0 = np.random.default_rng(1).normal(size=D)
        v0 = np.random.default_rng(2).normal(size=D)
        s0 = np.concatenate([x0, v0 + 0.5 * eps * m.grad(torch.as_tensor(x0, device="cuda")).cpu().numpy()])
        lf = cs.LeapfrogSystem(m, eps, L, dtype=torch.float64)
        ms, r = timed(lambda: cs.run_deer(lf, s0, cs.DeerConfig(mode="block2x2-stochastic")), 5)
        rows.append(("cfg4 leapfrog Gaussian D=1000 L=100 block (per proposal)", ms, r, L, None))
    if "4p" in which:
        # HMC with the parallel leapfrog inside each proposal at cfg 4's width: one
        # batched step_batch over B chain rows (every row's inner block solve)
        D, eps, L, B = 1000, 0.05, 100, 64
        m = cs.model_logp_grad_hvp(cs.gaussian(np.zeros(D), cfg4_chol(D)))
        S = torch.as_tensor(np.random.default_rng(1).normal(size=(B, D)), device="cuda")
        ts = torch.arange(1, B + 1, device="cuda")
        for eng in ("auto", "streamed"):
            k = cs.HmcKernel(m, eps, L, seed=3, T=B, leapfrog_mode="parallel",
                             leapfrog_cfg=cs.DeerConfig(mode="block2x2-stochastic", engine=eng))
            ms, _ = timed(lambda: k.step_batch(ts, S), 2)
            print(json.dumps({"config": f"cfg4 HMC parallel-leapfrog D=1000 L=100, step_batch over {B} rows",
                              "inner": "batched (one GEMM per pass for all rows)" if eng == "auto" else
                              "per-row run_deer (streamed)", "ms": round(ms, 3), "ms_per_proposal": round(ms / B, 3),
                              "fallbacks": len(k.fallback_events)}), flush=True)
    if "5" in which:
        k = cs.GibbsKernel(cs.generate_eight_schools(), seed=0, T=1_000_000, dtype=dt)
        s0 = k.initial_state()
        cfg = cs.DeerConfig(mode="diag-stochastic", hutchinson_samples=3, preconditioner=k.recommended_preconditioner(),
                            max_iters=400)
        ms, r = timed(lambda: cs.run_deer(k, s0, cfg), 3)
        rows.append(("cfg5 Gibbs eight schools T=1M diag x3 + precond", ms, r, 1_000_000, 808))
    for name, ms, r, T, cpu in rows:
        sps = T / (ms / 1e3)
        print(json.dumps({"config": name, "ms": round(ms, 3), "iterations": r.iterations, "converged": r.converged,
                          "samples_per_s": sps, "engine": r.stats.get("path"),
                          "reference_cpu_samples_per_s": cpu,
                          "speedup_vs_reference_cpu": (sps / cpu) if cpu else None}), flush=True)


if __name__ == "__main__":
    main()

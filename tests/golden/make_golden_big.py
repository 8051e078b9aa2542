"""Reference fixtures at the BASELINE.json sizes (cfg1 T=10K, cfg2 T=100K,
cfg3 diag T=100K, cfg4 D=1000 L=100, cfg5 T=1M), made by running the REFERENCE itself.

Run in the build container (the only place /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        CHAINSCAN_THREADS=8 python tests/golden/make_golden_big.py [cfg1 cfg2 cfg3 cfg4 cfg5]

The full traces are too large to commit, so each fixture keeps a compact but
size-independent record of the run: iterations, converged, the whole
delta_history, the whole per-step convergence record (int32), trace rows every
``stride`` steps, the sequential trace's rows at the same stride, the
sequential chain's accept mask (bit-packed: step t accepted iff s_t != s_{t-1})
and a few summary checksums.  Wall times of the reference runs are recorded
too (this container's 8 vCPUs, numba threads = CHAINSCAN_THREADS).
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

os.environ.setdefault("CHAINSCAN_THREADS", "8")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, "/root/reference/pkg/src")

from chainscan.core import sequential_evaluate  # noqa: E402
from chainscan.deer import DeerConfig, run_deer  # noqa: E402
from chainscan.samplers import GibbsKernel, HmcKernel, MalaKernel, generate_eight_schools  # noqa: E402
from chainscan.targets import blr, gaussian, model_logp_grad_hvp, rosenbrock, synthetic_credit_like  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
WORKERS = int(os.environ["CHAINSCAN_THREADS"])


def accept_bits(s0, seq):
    prev = np.concatenate([np.asarray(s0)[None], seq[:-1]], axis=0)
    return np.packbits(np.any(seq != prev, axis=1))


def record(out, prefix, res, stride, wall):
    out[prefix + "iterations"] = np.array(res.iterations)
    out[prefix + "converged"] = np.array(res.converged)
    out[prefix + "delta_history"] = np.asarray(res.delta_history)
    out[prefix + "psca"] = np.asarray(res.per_step_converged_at, dtype=np.int32)
    out[prefix + "rows"] = res.trace[stride - 1::stride].copy()
    out[prefix + "mean"] = res.trace.mean(axis=0)
    out[prefix + "wall_s"] = np.array(wall)


def seq_record(out, k, s0, stride):
    t0 = time.perf_counter()
    seq = sequential_evaluate(k, s0)
    out["seq_wall_s"] = np.array(time.perf_counter() - t0)
    out["seq_rows"] = seq[stride - 1::stride].copy()
    out["seq_accept_bits"] = accept_bits(s0, seq)
    out["seq_mean"] = seq.mean(axis=0)
    out["seq_last"] = seq[-1].copy()
    return seq


def timed_deer(k, s0, cfg):
    t0 = time.perf_counter()
    r = run_deer(k, s0, cfg)
    return r, time.perf_counter() - t0


def save(name, out):
    np.savez_compressed(os.path.join(OUT, name + ".npz"), **out)
    print("wrote", name, {k: np.asarray(v).shape for k, v in out.items()}, flush=True)


def cfg1():
    out = {"stride": np.array(20)}
    m = model_logp_grad_hvp(gaussian(np.array([1.0, -1.0]), np.array([[1.0, 0.0], [-0.6, 1.2]])))
    s0 = np.zeros(2)
    seq_record(out, MalaKernel(m, eps=0.4, seed=0, T=10_000), s0, 20)
    r, w = timed_deer(MalaKernel(m, eps=0.4, seed=0, T=10_000), s0, DeerConfig(mode="dense", workers=WORKERS))
    record(out, "dense_", r, 20, w)
    r, w = timed_deer(MalaKernel(m, eps=0.4, seed=0, T=10_000), s0,
                      DeerConfig(mode="dense", atol=1e-6, rtol=1e-5, workers=WORKERS))
    record(out, "tight_", r, 20, w)
    save("big_cfg1_mala_gauss2d_T10K", out)


def cfg2():
    out = {"stride": np.array(100)}
    m = model_logp_grad_hvp(rosenbrock(a=0.0, b=0.1, scale1=1.0, scale2=1.0))
    s0 = np.zeros(2)
    seq_record(out, HmcKernel(m, eps=0.5, L=8, seed=0, T=100_000), s0, 100)
    r, w = timed_deer(HmcKernel(m, eps=0.5, L=8, seed=0, T=100_000), s0,
                      DeerConfig(mode="diag-stochastic", clip=1.0, workers=WORKERS))
    record(out, "diagclip_", r, 100, w)
    save("big_cfg2_hmc_rosen2d_T100K", out)


def cfg3():
    out = {"stride": np.array(500)}
    X, y, _ = synthetic_credit_like(seed=20250819, n=1000, dim=100)
    m = model_logp_grad_hvp(blr(X, y, 1.0))
    s0 = np.zeros(100)
    seq_record(out, MalaKernel(m, eps=0.003, seed=4, T=100_000), s0, 500)
    r, w = timed_deer(MalaKernel(m, eps=0.003, seed=4, T=100_000), s0,
                      DeerConfig(mode="diag-stochastic", workers=WORKERS))
    record(out, "diag_", r, 500, w)
    save("big_cfg3_mala_blr100_T100K", out)


def cfg4():
    # the leapfrog trajectory inside one HMC proposal at full width: D = 1000
    # correlated Gaussian, L = 100, eps = 0.05, block vs diag
    from chainscan.samplers import LeapfrogSystem

    out = {"stride": np.array(10)}
    D = 1000
    rng = np.random.default_rng(0)
    Q, _ = np.linalg.qr(rng.normal(size=(D, D)))
    lam = np.exp(rng.uniform(np.log(0.1), np.log(10.0), D))
    Lc = np.linalg.cholesky((Q * lam) @ Q.T)
    m = model_logp_grad_hvp(gaussian(np.zeros(D), Lc))
    x0 = np.random.default_rng(1).normal(size=D)
    v0 = np.random.default_rng(2).normal(size=D)
    s0 = np.concatenate([x0, v0 + 0.5 * 0.05 * m.grad(x0)])
    lf = LeapfrogSystem(m, eps=0.05, L=100, probe_seed=0)
    out["s0"] = s0
    seq = sequential_evaluate(lf, s0)
    out["seq_rows"] = seq[9::10].copy()
    for mode, pre in (("block2x2-stochastic", "block_"), ("diag-stochastic", "diag_")):
        r, w = timed_deer(LeapfrogSystem(m, eps=0.05, L=100, probe_seed=0), s0, DeerConfig(mode=mode, workers=WORKERS))
        record(out, pre, r, 10, w)
    save("big_cfg4_leapfrog_gauss1000", out)


def cfg5():
    out = {"stride": np.array(2000)}
    data = generate_eight_schools()
    k = GibbsKernel(data, seed=0, T=1_000_000)
    s0 = k.initial_state()
    out["s0"] = s0
    seq_record(out, k, s0, 2000)
    cfg = DeerConfig(mode="diag-stochastic", hutchinson_samples=3,
                     preconditioner=k.recommended_preconditioner(), max_iters=400, workers=WORKERS)
    r, w = timed_deer(GibbsKernel(data, seed=0, T=1_000_000), s0, cfg)
    record(out, "diag3_", r, 2000, w)
    save("big_cfg5_gibbs_T1M", out)


if __name__ == "__main__":
    todo = sys.argv[1:] or ["cfg1", "cfg2", "cfg4", "cfg5", "cfg3"]
    for name in todo:
        t0 = time.perf_counter()
        globals()[name]()
        print(name, f"{time.perf_counter() - t0:.0f}s", flush=True)

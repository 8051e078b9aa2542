"""Generate golden vectors by running the REFERENCE implementation itself.

Run in the build container (the only place /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        CHAINSCAN_THREADS=4 python tests/golden/make_golden.py

Writes ``tests/golden/*.npz``.  The fixtures pin the CPU oracle (``oracle/``)
and, through it, the CUDA product.  Nothing at test or bench time reads
/root/reference; only these committed files travel.
"""

from __future__ import annotations

import os
import sys

import numpy as np

os.environ.setdefault("CHAINSCAN_THREADS", "4")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, "/root/reference/pkg/src")

from chainscan import noise as rnoise  # noqa: E402
from chainscan import pscan as rpscan  # noqa: E402
from chainscan.core import sequential_evaluate  # noqa: E402
from chainscan.deer import DeerConfig, run_deer  # noqa: E402
from chainscan.samplers import (  # noqa: E402
    GibbsKernel,
    HmcKernel,
    LeapfrogSystem,
    MalaKernel,
    generate_eight_schools,
)
from chainscan.targets import (  # noqa: E402
    blr,
    gaussian,
    model_logp_grad_hvp,
    mog,
    rosenbrock,
    std_normal,
    synthetic_credit_like,
)

OUT = os.path.dirname(os.path.abspath(__file__))
WORKERS = 4


def save(name, **arrays):
    np.savez_compressed(os.path.join(OUT, name + ".npz"), **arrays)
    print("wrote", name, {k: np.asarray(v).shape for k, v in arrays.items()})


def noise_fixtures():
    layout = {
        "xi": rnoise.SlotSpec(3, "standard-normal"),
        "u": rnoise.SlotSpec(1, "uniform-0-1"),
        "g": rnoise.SlotSpec(2, "chi-squared", df=9.1),
        "g_small": rnoise.SlotSpec(2, "chi-squared", df=0.1),
        "g_big": rnoise.SlotSpec(8, "chi-squared", df=20.1),
    }
    tab = rnoise.NoiseTable(7, layout, T=300)
    ts = np.arange(301)
    out = {k: tab.block(k, ts) for k in layout}
    out["slot_ids"] = np.array([rnoise._fnv1a(k) for k in layout], dtype=np.uint64)
    out["hash"] = rnoise._counter_hash(
        123456789, np.arange(5, dtype=np.uint64)[:, None], 17, np.arange(7, dtype=np.uint64)[None, :])
    big = rnoise.NoiseTable(2**63 + 12345, {"xi": rnoise.SlotSpec(2, "standard-normal")}, T=10)
    out["xi_bigseed"] = big.block("xi", np.arange(11))
    probes = []
    for it in range(3):
        for k in range(3):
            probes.append(rnoise.rademacher_probe(9, it, np.arange(1, 65), k, 6))
    out["probes"] = np.stack(probes)
    save("noise", **out)


def scan_fixtures():
    rng = np.random.default_rng(2025)
    out = {}
    for T in (1, 257, 1024):
        D = 4
        j = rng.uniform(-0.9, 0.9, (T, D)); u = rng.normal(size=(T, D)); s0 = rng.normal(size=D)
        out[f"diag_{T}_j"], out[f"diag_{T}_u"], out[f"diag_{T}_s0"] = j, u, s0
        out[f"diag_{T}_out"] = rpscan.parallel_affine_solve(rpscan.DiagElements(j, u), s0, workers=WORKERS)
        out[f"diag_{T}_out_c128"] = rpscan.parallel_affine_solve(rpscan.DiagElements(j, u), s0, workers=WORKERS, chunk=128)
        J = rng.normal(size=(T, D, D))
        J *= (0.9 / np.abs(np.linalg.eigvals(J)).max(axis=-1))[:, None, None]
        u = rng.normal(size=(T, D)); s0 = rng.normal(size=D)
        out[f"dense_{T}_J"], out[f"dense_{T}_u"], out[f"dense_{T}_s0"] = J, u, s0
        out[f"dense_{T}_out"] = rpscan.parallel_affine_solve(rpscan.DenseElements(J, u), s0, workers=WORKERS)
        a, b, c, d = (rng.uniform(-0.9, 0.9, (T, D)) for _ in range(4))
        u = rng.normal(size=(T, 2 * D)); s0 = rng.normal(size=2 * D)
        for nm, arr in zip("abcd", (a, b, c, d)):
            out[f"block_{T}_{nm}"] = arr
        out[f"block_{T}_u"], out[f"block_{T}_s0"] = u, s0
        out[f"block_{T}_out"] = rpscan.parallel_affine_solve(
            rpscan.Block2x2Elements(a, b, c, d, u), s0, workers=WORKERS)
    save("scan", **out)


def deer_record(prefix, res, out):
    out[prefix + "trace"] = res.trace
    out[prefix + "iterations"] = np.array(res.iterations)
    out[prefix + "delta_history"] = np.asarray(res.delta_history)
    out[prefix + "converged"] = np.array(res.converged)
    out[prefix + "psca"] = np.asarray(res.per_step_converged_at)


def chain_fixtures():
    # cfg1 (reduced T): MALA on the criterion-8 Gaussian, dense and diag
    out = {}
    m = model_logp_grad_hvp(gaussian(np.array([1.0, -1.0]), np.array([[1.0, 0.0], [-0.6, 1.2]])))
    k = MalaKernel(m, eps=0.4, seed=0, T=2000)
    s0 = np.zeros(2)
    out["seq"] = sequential_evaluate(k, s0)
    deer_record("dense_", run_deer(k, s0, DeerConfig(mode="dense", workers=WORKERS)), out)
    deer_record("diag_", run_deer(k, s0, DeerConfig(mode="diag-stochastic", workers=WORKERS)), out)
    deer_record("tight_", run_deer(k, s0, DeerConfig(mode="dense", atol=1e-6, rtol=1e-5, workers=WORKERS)), out)
    save("mala_gauss2d", **out)

    out = {}
    m = model_logp_grad_hvp(rosenbrock(b=0.1, scale2=1.0))
    k = MalaKernel(m, eps=0.5, seed=0, T=2000)
    out["seq"] = sequential_evaluate(k, s0)
    deer_record("dense_", run_deer(k, s0, DeerConfig(mode="dense", workers=WORKERS)), out)
    save("mala_rosen2d", **out)

    # cfg2 (reduced T): HMC on the gentle Rosenbrock, diag + clip
    out = {}
    m = model_logp_grad_hvp(rosenbrock(a=0.0, b=0.1, scale1=1.0, scale2=1.0))
    k = HmcKernel(m, eps=0.5, L=8, seed=0, T=5000)
    out["seq"] = sequential_evaluate(k, s0)
    deer_record("diagclip_", run_deer(k, s0, DeerConfig(mode="diag-stochastic", clip=1.0, workers=WORKERS)), out)
    deer_record("dense_", run_deer(k, s0, DeerConfig(mode="dense", damping=0.5, clip=1.0, atol=1e-6, rtol=1e-5, workers=WORKERS)), out)
    save("hmc_rosen2d", **out)

    # MoG MALA with damping (secondary target)
    out = {}
    m = model_logp_grad_hvp(mog())
    k = MalaKernel(m, eps=0.1, seed=3, T=1000)
    out["seq"] = sequential_evaluate(k, s0)
    deer_record("damped_", run_deer(k, s0, DeerConfig(mode="diag-stochastic", damping=0.5, max_iters=300, workers=WORKERS)), out)
    save("mala_mog2d", **out)

    # cfg3 (reduced T): BLR MALA on the synthetic credit data, D=100
    out = {}
    X, y, beta = synthetic_credit_like(seed=20250819, n=1000, dim=100)
    out["X"], out["y"], out["beta_star"] = X, y, beta
    m = model_logp_grad_hvp(blr(X, y, 1.0))
    k = MalaKernel(m, eps=0.003, seed=4, T=300)
    s0 = np.zeros(100)
    out["seq"] = sequential_evaluate(k, s0)
    deer_record("diag_", run_deer(k, s0, DeerConfig(mode="diag-stochastic", workers=WORKERS)), out)
    save("mala_blr100", **out)

    # cfg4 (reduced D): leapfrog on a correlated Gaussian, block vs diag
    out = {}
    D = 200
    rng = np.random.default_rng(0)
    Q, _ = np.linalg.qr(rng.normal(size=(D, D)))
    lam = np.exp(rng.uniform(np.log(0.1), np.log(10.0), D))
    P = (Q * lam) @ Q.T
    Lc = np.linalg.cholesky(P)
    m = model_logp_grad_hvp(gaussian(np.zeros(D), Lc))
    out["chol"] = Lc
    lf = LeapfrogSystem(m, eps=0.05, L=100, probe_seed=0)
    x0 = np.random.default_rng(1).normal(size=D)
    v0 = np.random.default_rng(2).normal(size=D)
    s0 = np.concatenate([x0, v0 + 0.5 * 0.05 * m.grad(x0)])
    out["s0"] = s0
    out["seq"] = sequential_evaluate(lf, s0)
    deer_record("block_", run_deer(lf, s0, DeerConfig(mode="block2x2-stochastic", workers=WORKERS)), out)
    deer_record("diag_", run_deer(lf, s0, DeerConfig(mode="diag-stochastic", workers=WORKERS)), out)
    save("leapfrog_gauss200", **out)

    # cfg5 (reduced T): eight-schools Gibbs, diag x3 + preconditioner
    out = {}
    data = generate_eight_schools()
    out["x"] = data.x
    k = GibbsKernel(data, seed=0, T=3000)
    s0 = k.initial_state()
    out["s0"] = s0
    out["seq"] = sequential_evaluate(k, s0)
    cfg = DeerConfig(mode="diag-stochastic", hutchinson_samples=3,
                     preconditioner=k.recommended_preconditioner(), max_iters=400, workers=WORKERS)
    deer_record("diag3_", run_deer(k, s0, cfg), out)
    save("gibbs_schools", **out)

    # HMC with the inner parallel leapfrog solve
    out = {}
    m = model_logp_grad_hvp(rosenbrock(b=0.1, scale2=1.0))
    k = HmcKernel(m, eps=0.2, L=16, seed=5, T=40, leapfrog_mode="parallel",
                  leapfrog_cfg=DeerConfig(mode="block2x2-stochastic", workers=WORKERS))
    out["seq"] = sequential_evaluate(k, np.array([0.5, -0.5]))
    out["fallbacks"] = np.array(k.fallback_events, dtype=np.int64).reshape(-1, 2)
    save("hmc_parallel_leapfrog", **out)

    # sliding window on std-normal MALA
    out = {}
    m = model_logp_grad_hvp(std_normal(2))
    k = MalaKernel(m, eps=0.3, seed=6, T=512)
    s0 = np.array([1.0, 0.0])
    deer_record("win64_", run_deer(k, s0, DeerConfig(mode="dense", window_len=64, max_iters=2000, workers=WORKERS)), out)
    deer_record("win1_", run_deer(MalaKernel(m, eps=0.3, seed=6, T=40), s0,
                                  DeerConfig(mode="dense", window_len=1, max_iters=500, workers=WORKERS)), out)
    save("mala_window", **out)


def blr_dense_fixture():
    # cfg3 "full" (reduced T): the same BLR MALA chain as mala_blr100, solved
    # with dense (full-Jacobian) Newton -- D = 100, the wide dense scan
    out = {}
    X, y, _ = synthetic_credit_like(seed=20250819, n=1000, dim=100)
    m = model_logp_grad_hvp(blr(X, y, 1.0))
    k = MalaKernel(m, eps=0.003, seed=4, T=300)
    deer_record("dense_", run_deer(k, np.zeros(100), DeerConfig(mode="dense", workers=WORKERS)), out)
    save("mala_blr100_dense", **out)


def trace_fixture():
    # the reference's own trace artifact (tracefile.py): payload + sidecar + CSV
    from chainscan.tracefile import export_csv, write_trace

    rng = np.random.default_rng(17)
    tr = rng.normal(size=(2, 5, 3))
    tr[0, 0, 0], tr[1, 4, 2] = 1e-300, -np.inf
    base = os.path.join(OUT, "trace_ref.bin")
    write_trace(base, tr, "hmc", 123, {"eps": 0.5, "L": 8, "method": "quasi-deer"})
    export_csv(os.path.join(OUT, "trace_ref.csv"), tr)
    np.save(os.path.join(OUT, "trace_ref_array.npy"), tr)
    print("wrote trace_ref")


def basis_fixture():
    # orthogonal change of basis (targets.py:400-517): Jacobi eigenbasis of a random
    # symmetric matrix, and a diag quasi-Newton MALA solve in the eigenbasis of a
    # correlated Gaussian's precision
    from chainscan.targets import orthogonal_basis, transform_system

    out = {}
    rng = np.random.default_rng(5)
    M = rng.normal(size=(16, 16))
    C = M + M.T
    b = orthogonal_basis(C)
    out["C"], out["Q"], out["eig"] = C, b.Q, b.eigenvalues
    A = rng.normal(size=(4, 4))
    P = A @ A.T + 0.5 * np.eye(4)
    Lc = np.linalg.cholesky(P)
    m = model_logp_grad_hvp(gaussian(np.array([0.5, -1.0, 0.0, 1.0]), Lc))
    k = MalaKernel(m, eps=0.15, seed=9, T=400)
    basis = orthogonal_basis(P)
    w = transform_system(k, basis.Q)
    s0 = np.zeros(4)
    out["chol"], out["P"], out["Qp"] = Lc, P, basis.Q
    r = run_deer(w, w.transform_state(s0), DeerConfig(mode="diag-stochastic", workers=WORKERS))
    out["z_trace"], out["z_iterations"], out["z_converged"] = r.trace, np.array(r.iterations), np.array(r.converged)
    out["seq"] = sequential_evaluate(k, s0)
    r2 = run_deer(k, s0, DeerConfig(mode="diag-stochastic", workers=WORKERS))
    out["plain_iterations"] = np.array(r2.iterations)
    save("basis", **out)


if __name__ == "__main__":
    if sys.argv[1:] == ["basis"]:
        basis_fixture()
        sys.exit(0)
    if sys.argv[1:] == ["blr_dense"]:
        blr_dense_fixture()
        sys.exit(0)
    if sys.argv[1:] == ["trace"]:
        trace_fixture()
        sys.exit(0)
    noise_fixtures()
    scan_fixtures()
    chain_fixtures()
    blr_dense_fixture()
    trace_fixture()
    basis_fixture()

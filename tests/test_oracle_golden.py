"""Pin the CPU oracle to golden vectors produced by the reference itself.

The fixtures come from ``tests/golden/make_golden.py`` (run against
/root/reference in the build container).  With the same chunk layout
(``workers=4``) the oracle must reproduce the reference's f64 outputs exactly
or to a few ulp; these are CPU tests (``-m "not gpu"``).
"""

import numpy as np
import pytest

import oracle as O
from oracle.systems import HYPER
from conftest import golden

W = 4


def _check_deer(res, g, prefix, exact=True):
    assert res.iterations == int(g[prefix + "iterations"])
    assert res.converged == bool(g[prefix + "converged"])
    np.testing.assert_array_equal(res.per_step_converged_at, g[prefix + "psca"])
    if exact:
        np.testing.assert_array_equal(res.trace, g[prefix + "trace"])
        np.testing.assert_array_equal(res.delta_history, g[prefix + "delta_history"])
    else:
        np.testing.assert_allclose(res.trace, g[prefix + "trace"], atol=1e-10, rtol=0)
        np.testing.assert_allclose(res.delta_history, g[prefix + "delta_history"], rtol=1e-8, atol=1e-12)


def test_noise_golden():
    g = golden("noise")
    layout = {"xi": O.SlotSpec(3, "standard-normal"), "u": O.SlotSpec(1, "uniform-0-1"),
              "g": O.SlotSpec(2, "chi-squared", df=9.1),
              "g_small": O.SlotSpec(2, "chi-squared", df=0.1),
              "g_big": O.SlotSpec(8, "chi-squared", df=20.1)}
    tab = O.NoiseTable(7, layout, 300)
    for k in layout:
        np.testing.assert_array_equal(tab.block(k, np.arange(301)), g[k])
    np.testing.assert_array_equal(np.array([O.fnv1a64(k) for k in layout], dtype=np.uint64), g["slot_ids"])
    h = O.counter_hash(123456789, np.arange(5, dtype=np.uint64)[:, None], 17,
                       np.arange(7, dtype=np.uint64)[None, :])
    np.testing.assert_array_equal(h, g["hash"])
    big = O.NoiseTable(2**63 + 12345, {"xi": O.SlotSpec(2, "standard-normal")}, 10)
    np.testing.assert_array_equal(big.block("xi", np.arange(11)), g["xi_bigseed"])
    probes = [O.rademacher_probe(9, it, np.arange(1, 65), k, 6) for it in range(3) for k in range(3)]
    np.testing.assert_array_equal(np.stack(probes), g["probes"])


@pytest.mark.parametrize("T", [1, 257, 1024])
def test_scan_golden(T):
    g = golden("scan")
    d = O.DiagElements(g[f"diag_{T}_j"], g[f"diag_{T}_u"])
    np.testing.assert_array_equal(O.parallel_affine_solve(d, g[f"diag_{T}_s0"], workers=W), g[f"diag_{T}_out"])
    np.testing.assert_array_equal(O.parallel_affine_solve(d, g[f"diag_{T}_s0"], workers=W, chunk=128),
                                  g[f"diag_{T}_out_c128"])
    e = O.DenseElements(g[f"dense_{T}_J"], g[f"dense_{T}_u"])
    np.testing.assert_array_equal(O.parallel_affine_solve(e, g[f"dense_{T}_s0"], workers=W), g[f"dense_{T}_out"])
    b = O.Block2x2Elements(*(g[f"block_{T}_{k}"] for k in "abcdu"))
    np.testing.assert_array_equal(O.parallel_affine_solve(b, g[f"block_{T}_s0"], workers=W), g[f"block_{T}_out"])
    for el, key in ((d, "diag"), (e, "dense"), (b, "block")):
        np.testing.assert_allclose(O.sequential_affine_solve(el, g[f"{key}_{T}_s0"]), g[f"{key}_{T}_out"],
                                   atol=1e-10)


def test_scan_kats():
    # test_pscan.py:55-62 and SPEC.md:119
    e = O.DiagElements(np.array([[2.0], [3.0], [4.0]]), np.ones((3, 1)))
    np.testing.assert_array_equal(O.parallel_affine_solve(e, np.array([1.0]))[:, 0], [3.0, 10.0, 41.0])
    # test_pscan.py:65-72
    e1 = O.DenseElements(np.array([[0.0, 1.0], [1.0, 0.0]]), np.array([1.0, 0.0]))
    e2 = O.DenseElements(2.0 * np.eye(2), np.zeros(2))
    c = O.compose(e2, e1)
    np.testing.assert_array_equal(c.J, [[0.0, 2.0], [2.0, 0.0]])
    np.testing.assert_array_equal(c.u, [2.0, 0.0])
    # test_pscan.py:200-203
    assert O.default_chunk(100, 4) == 100
    assert O.default_chunk(10_000, 4) == 313
    assert O.default_chunk(1_000_000, 8) == 15625
    # test_deer.py:305-308
    assert O.default_max_iters(256) == 51
    assert O.default_max_iters(10_000) == 55
    assert O.default_max_iters(1_000_000) == 550


def test_mala_gauss2d_golden():
    g = golden("mala_gauss2d")
    m = O.gaussian([1.0, -1.0], [[1.0, 0.0], [-0.6, 1.2]])
    k = O.MalaKernel(m, 0.4, seed=0, T=2000)
    np.testing.assert_array_equal(O.sequential_evaluate(k, np.zeros(2)), g["seq"])
    _check_deer(O.run_deer(k, np.zeros(2), O.DeerConfig(mode="dense", workers=W)), g, "dense_")
    _check_deer(O.run_deer(k, np.zeros(2), O.DeerConfig(mode="diag-stochastic", workers=W)), g, "diag_")
    _check_deer(O.run_deer(k, np.zeros(2), O.DeerConfig(mode="dense", atol=1e-6, rtol=1e-5, workers=W)),
                g, "tight_")


def test_mala_rosen2d_golden():
    g = golden("mala_rosen2d")
    k = O.MalaKernel(O.rosenbrock(b=0.1, scale2=1.0), 0.5, seed=0, T=2000)
    np.testing.assert_array_equal(O.sequential_evaluate(k, np.zeros(2)), g["seq"])
    _check_deer(O.run_deer(k, np.zeros(2), O.DeerConfig(mode="dense", workers=W)), g, "dense_")


def test_hmc_rosen2d_golden():
    g = golden("hmc_rosen2d")
    k = O.HmcKernel(O.rosenbrock(a=0.0, b=0.1, scale1=1.0, scale2=1.0), 0.5, 8, seed=0, T=5000)
    np.testing.assert_array_equal(O.sequential_evaluate(k, np.zeros(2)), g["seq"])
    _check_deer(O.run_deer(k, np.zeros(2), O.DeerConfig(mode="diag-stochastic", clip=1.0, workers=W)),
                g, "diagclip_")
    _check_deer(O.run_deer(k, np.zeros(2), O.DeerConfig(mode="dense", damping=0.5, clip=1.0, atol=1e-6,
                                                        rtol=1e-5, workers=W)), g, "dense_")


def test_mala_mog_golden():
    g = golden("mala_mog2d")
    k = O.MalaKernel(O.mog(), 0.1, seed=3, T=1000)
    np.testing.assert_array_equal(O.sequential_evaluate(k, np.zeros(2)), g["seq"])
    _check_deer(O.run_deer(k, np.zeros(2), O.DeerConfig(mode="diag-stochastic", damping=0.5, max_iters=300,
                                                        workers=W)), g, "damped_")


def test_blr_golden():
    g = golden("mala_blr100")
    X, y, beta = O.synthetic_credit_like(seed=20250819, n=1000, dim=100)
    np.testing.assert_array_equal(X, g["X"])
    np.testing.assert_array_equal(y, g["y"])
    np.testing.assert_array_equal(beta, g["beta_star"])
    k = O.MalaKernel(O.blr(X, y, 1.0), 0.003, seed=4, T=300)
    np.testing.assert_allclose(O.sequential_evaluate(k, np.zeros(100)), g["seq"], atol=1e-12, rtol=0)
    _check_deer(O.run_deer(k, np.zeros(100), O.DeerConfig(mode="diag-stochastic", workers=W)), g, "diag_",
                exact=False)


def test_blr_dense_golden():
    # cfg3 "full": dense Newton at D = 100 (the reference's D-jvp Jacobian)
    g0, g = golden("mala_blr100"), golden("mala_blr100_dense")
    k = O.MalaKernel(O.blr(g0["X"], g0["y"], 1.0), 0.003, seed=4, T=300)
    _check_deer(O.run_deer(k, np.zeros(100), O.DeerConfig(mode="dense", workers=W)), g, "dense_", exact=False)


def test_leapfrog_gauss_golden():
    g = golden("leapfrog_gauss200")
    D = 200
    m = O.gaussian(np.zeros(D), g["chol"])
    lf = O.LeapfrogSystem(m, 0.05, 100, probe_seed=0)
    np.testing.assert_allclose(O.sequential_evaluate(lf, g["s0"]), g["seq"], atol=1e-12, rtol=0)
    _check_deer(O.run_deer(lf, g["s0"], O.DeerConfig(mode="block2x2-stochastic", workers=W)), g, "block_",
                exact=False)
    _check_deer(O.run_deer(lf, g["s0"], O.DeerConfig(mode="diag-stochastic", workers=W)), g, "diag_",
                exact=False)


def test_gibbs_golden():
    g = golden("gibbs_schools")
    data = O.generate_eight_schools()
    np.testing.assert_array_equal(data.x, g["x"])
    k = O.GibbsKernel(data, seed=0, T=3000)
    s0 = k.initial_state()
    np.testing.assert_array_equal(s0, g["s0"])
    np.testing.assert_array_equal(O.sequential_evaluate(k, s0), g["seq"])
    cfg = O.DeerConfig(mode="diag-stochastic", hutchinson_samples=3,
                       preconditioner=k.recommended_preconditioner(), max_iters=400, workers=W)
    _check_deer(O.run_deer(k, s0, cfg), g, "diag3_")
    assert HYPER["nu0"] == 0.1


def test_hmc_parallel_leapfrog_golden():
    g = golden("hmc_parallel_leapfrog")
    k = O.HmcKernel(O.rosenbrock(b=0.1, scale2=1.0), 0.2, 16, seed=5, T=40, leapfrog_mode="parallel",
                    leapfrog_cfg=O.DeerConfig(mode="block2x2-stochastic", workers=W))
    np.testing.assert_allclose(O.sequential_evaluate(k, np.array([0.5, -0.5])), g["seq"], atol=1e-12, rtol=0)
    assert len(k.fallback_events) == len(g["fallbacks"])


def test_window_golden():
    g = golden("mala_window")
    m = O.std_normal(2)
    k = O.MalaKernel(m, 0.3, seed=6, T=512)
    _check_deer(O.run_deer(k, np.array([1.0, 0.0]),
                           O.DeerConfig(mode="dense", window_len=64, max_iters=2000, workers=W)), g, "win64_")
    _check_deer(O.run_deer(O.MalaKernel(m, 0.3, seed=6, T=40), np.array([1.0, 0.0]),
                           O.DeerConfig(mode="dense", window_len=1, max_iters=500, workers=W)), g, "win1_")

"""Kernel-level checks mirrored from the reference's tests/test_samplers.py
(TestLeapfrog, TestHmc, TestGibbs) against this package's samplers: every
expected value comes from a straight-line reimplementation (Stormer-Verlet
with explicit half-kicks, Hamiltonians recomputed from the noise table), not
from the kernels themselves."""

import numpy as np
import pytest
import torch

import paper_2508_18413_b200 as cs
from paper_2508_18413_b200.errors import ChainDivergedError, ConfigurationError
from paper_2508_18413_b200.samplers import (CLASSIC_EFFECTS, CLASSIC_SES, gibbs_sweep, hmc_chain_system, hmc_step,
                                            leapfrog_block_jacobian, leapfrog_step)

pytestmark = pytest.mark.gpu


def np_(x):
    return x.detach().cpu().numpy() if torch.is_tensor(x) else np.asarray(x)


def t64(x):
    return torch.as_tensor(np.asarray(x, float), dtype=torch.float64, device="cuda")


def grad(model, x):
    return np_(model.grad(t64(x)))


def verlet(model, x, v, eps, L, mass=None):
    """Symplectic trajectory with explicit half-kicks at both ends (test_samplers.py:64-73)."""
    mass = np.ones_like(x) if mass is None else np.asarray(mass, float)
    v = v + 0.5 * eps * grad(model, x)
    for k in range(L):
        x = x + eps * v / mass
        if k < L - 1:
            v = v + eps * grad(model, x)
    v = v + 0.5 * eps * grad(model, x)
    return x, v


def hamiltonian(model, x, v, mass=None):
    mass = np.ones_like(x) if mass is None else np.asarray(mass, float)
    return 0.5 * float(np.sum(v * v / mass)) - float(np_(model.logp(t64(x))))


# ---- leapfrog (test_samplers.py:193-307)
def test_single_step_from_rest(cuda_device):
    system = cs.LeapfrogSystem(cs.model_logp_grad_hvp(cs.std_normal(2)), 0.1, 8)
    out = np_(leapfrog_step(np.array([1.0, 0.0, 0.0, 0.0]), system))
    np.testing.assert_allclose(out[:2], [1.0, 0.0], atol=1e-15)
    np.testing.assert_allclose(out[2:], [-0.1, 0.0], atol=1e-15)


def test_step_via_hmc_kernel_matches_system(cuda_device):
    model = cs.model_logp_grad_hvp(cs.std_normal(2))
    s = np.array([0.3, -0.8, 0.5, 1.1])
    np.testing.assert_allclose(np_(leapfrog_step(s, cs.HmcKernel(model, 0.1, 8, seed=0, T=2))),
                               np_(leapfrog_step(s, cs.LeapfrogSystem(model, 0.1, 8))), atol=1e-15)


def test_symmetric_trajectory_is_time_reversible(cuda_device):
    model = cs.model_logp_grad_hvp(cs.std_normal(2))
    x0, v0 = np.array([1.3, -0.7]), np.array([0.4, 0.9])
    xl, vl = verlet(model, x0, v0, 0.1, 16)
    xb, vb = verlet(model, xl, -vl, 0.1, 16)
    np.testing.assert_allclose(xb, x0, atol=1e-10)
    np.testing.assert_allclose(vb, -v0, atol=1e-10)


def test_staggered_steps_compose_into_the_symmetric_trajectory(cuda_device):
    model = cs.model_logp_grad_hvp(cs.std_normal(2))
    eps, L = 0.1, 16
    x0, v0 = np.array([1.3, -0.7]), np.array([0.4, 0.9])
    system = cs.LeapfrogSystem(model, eps, L)
    s = np.concatenate([x0, v0 + 0.5 * eps * grad(model, x0)])
    for _ in range(L):
        s = np_(leapfrog_step(s, system))
    x, v = s[:2], s[2:] - 0.5 * eps * grad(model, s[:2])
    xl, vl = verlet(model, x0, v0, eps, L)
    np.testing.assert_allclose(x, xl, atol=1e-13)
    np.testing.assert_allclose(v, vl, atol=1e-13)


def test_energy_drift_stays_small(cuda_device):
    model = cs.model_logp_grad_hvp(cs.std_normal(2))
    x, v = np.array([1.2, -0.4]), np.array([0.3, 0.8])
    xl, vl = verlet(model, x, v, 0.01, 100)
    assert abs(hamiltonian(model, xl, vl) - hamiltonian(model, x, v)) <= 1e-4


@pytest.mark.parametrize("spec", ["gauss", "rosen"])
def test_volume_preserved(cuda_device, spec):
    tgt = cs.gaussian(np.zeros(2), np.array([[1.1, 0.0], [0.3, 0.8]])) if spec == "gauss" else cs.rosenbrock()
    system = cs.LeapfrogSystem(cs.model_logp_grad_hvp(tgt), 0.2, 4)
    rng = np.random.default_rng(5)
    for _ in range(3):
        s = rng.normal(size=4)
        J = np.column_stack([np_(system.jvp(1, s, e)) for e in np.eye(4)])
        assert abs(np.linalg.det(J) - 1.0) < 1e-10


def test_block_jacobian_exact_on_standard_normal(cuda_device):
    eps = 0.15
    system = cs.LeapfrogSystem(cs.model_logp_grad_hvp(cs.std_normal(3)), eps, 4)
    a, b, c, d = (np_(x) for x in leapfrog_block_jacobian(np.array([0.5, -1.0, 2.0, 0.2, 0.1, -0.3]), system, 1))
    np.testing.assert_allclose(a, np.ones(3), atol=1e-14)
    np.testing.assert_allclose(b, np.full(3, eps), atol=1e-14)
    np.testing.assert_allclose(c, np.full(3, -eps), atol=1e-14)
    np.testing.assert_allclose(d, np.full(3, 1 - eps * eps), atol=1e-14)


def test_block_matches_dense_jacobian_for_diagonal_hessian(cuda_device):
    prec = np.array([2.0, 0.5])
    system = cs.LeapfrogSystem(cs.model_logp_grad_hvp(cs.gaussian(np.zeros(2), np.diag(np.sqrt(prec)))), 0.1, 4)
    s = np.array([0.7, -0.2, 0.4, 1.5])
    a, b, c, d = (np_(x).ravel() for x in leapfrog_block_jacobian(s, system, 1))
    expected = np.block([[np.diag(a), np.diag(b)], [np.diag(c), np.diag(d)]])
    dense = np.column_stack([np_(system.jvp(1, s, e)) for e in np.eye(4)])
    np.testing.assert_allclose(expected, dense, atol=1e-12)


def test_rejects_bad_geometry(cuda_device):
    model = cs.model_logp_grad_hvp(cs.std_normal(2))
    for kw in (dict(eps=-0.1, L=4), dict(eps=0.1, L=0), dict(eps=0.1, L=4, mass=np.array([1.0, -1.0]))):
        with pytest.raises(ConfigurationError):
            cs.LeapfrogSystem(model, **kw)


# ---- HMC (test_samplers.py:310-390)
def test_gate_agrees_with_recomputed_hamiltonians(cuda_device):
    model = cs.model_logp_grad_hvp(cs.std_normal(3))
    mass = np.array([2.0, 0.5, 1.0])
    eps, L, T = 0.65, 5, 300
    kernel = cs.HmcKernel(model, eps, L, seed=7, T=T, mass=mass)
    x0 = np.array([1.5, -0.5, 2.0])
    trace = np_(cs.sequential_evaluate(kernel, x0))
    x, n_rejects, n_gains = x0, 0, 0
    for t in range(1, T + 1):
        xi = np_(kernel.noise.block("momentum", [t]))[0]
        u = np_(kernel.noise.block("u", [t]))[0, 0]
        v0 = np.sqrt(mass) * xi
        xl, vl = verlet(model, x, v0, eps, L, mass)
        delta = hamiltonian(model, x, v0, mass) - hamiltonian(model, xl, vl, mass)
        accept = np.log(u) < min(0.0, delta)
        if delta > 0:
            n_gains += 1
            assert accept
        if accept:
            np.testing.assert_allclose(trace[t - 1], xl, rtol=1e-10, atol=1e-12)
            x = trace[t - 1]
        else:
            n_rejects += 1
            assert np.array_equal(trace[t - 1], x)
    assert n_rejects > 10 and n_gains > 10


def test_parallel_leapfrog_matches_sequential(cuda_device):
    model = cs.model_logp_grad_hvp(cs.std_normal(2))
    x0 = np.array([1.5, -0.5])
    seq = hmc_chain_system(model, eps=0.1, L=32, seed=4, T=64)
    par = hmc_chain_system(model, eps=0.1, L=32, seed=4, T=64, leapfrog_mode="parallel")
    a, b = np_(cs.sequential_evaluate(seq, x0)), np_(cs.sequential_evaluate(par, x0))
    np.testing.assert_allclose(a, b, atol=1e-6)
    assert par.n_leapfrog_fallbacks == 0
    moved_a = np.any(np.diff(np.vstack([x0, a]), axis=0) != 0, axis=1)
    moved_b = np.any(np.abs(np.diff(np.vstack([x0, b]), axis=0)) > 1e-9, axis=1)
    assert np.array_equal(moved_a, moved_b)


def test_mode_override_wrapper(cuda_device):
    kernel = hmc_chain_system(cs.model_logp_grad_hvp(cs.std_normal(2)), eps=0.1, L=16, seed=8, T=4)
    x = np.array([0.9, -1.4])
    np.testing.assert_allclose(np_(hmc_step(x, 1, kernel)), np_(hmc_step(x, 1, kernel, leapfrog_mode="parallel")),
                               atol=1e-8)


def test_inner_solver_failure_falls_back_to_sequential(cuda_device):
    model = cs.model_logp_grad_hvp(cs.rosenbrock())
    cfg = cs.DeerConfig(mode="block2x2-stochastic", max_iters=1)
    par = hmc_chain_system(model, eps=0.05, L=16, seed=8, T=4, leapfrog_mode="parallel", leapfrog_cfg=cfg)
    seq = hmc_chain_system(model, eps=0.05, L=16, seed=8, T=4)
    x = np.array([0.9, -1.4])
    out = hmc_step(x, 1, par)
    assert par.n_leapfrog_fallbacks >= 1 and par.fallback_events[0][0] == 1
    np.testing.assert_allclose(np_(out), np_(hmc_step(x, 1, seq)), atol=1e-14)


# ---- Gibbs (test_samplers.py:590-640)
def test_initial_state_is_prior_draw_plus_one_sweep(cuda_device):
    kernel = cs.GibbsKernel(cs.generate_eight_schools(), seed=13, T=4)
    h = kernel.hyper
    blk = lambda name: np_(kernel.noise.block(name, [0]))[0]
    g_tau = blk("g_tau_prior")[0]
    tau2 = h.nu0 * h.tau0_sq / g_tau
    mu = h.mu0 + np.sqrt(tau2 / h.kappa0) * blk("xi_mu_prior")[0]
    theta = mu + np.sqrt(tau2) * blk("xi_theta_prior")
    sig2 = h.alpha0 * h.sigma0_sq / blk("g_sigma_prior")
    prior = np.concatenate([[tau2], [mu], theta, sig2])
    np.testing.assert_allclose(np_(kernel.initial_state()), np_(gibbs_sweep(prior, 0, kernel)), rtol=1e-12)


def test_initial_state_is_reproducible(cuda_device):
    data = cs.generate_eight_schools()
    a, b = np_(cs.GibbsKernel(data, seed=13, T=4).initial_state()), np_(cs.GibbsKernel(data, seed=13, T=4).initial_state())
    c = np_(cs.GibbsKernel(data, seed=14, T=4).initial_state())
    assert np.array_equal(a, b) and not np.array_equal(a, c)


def test_generated_data_reproduces_the_classic_table(cuda_device):
    data = cs.generate_eight_schools()
    n = data.n_per_school
    np.testing.assert_allclose(np_(data.xbar), CLASSIC_EFFECTS, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(np_(data.ss), (n - 1) * n * np.asarray(CLASSIC_SES) ** 2, rtol=1e-9)
    assert np.array_equal(np_(data.x), np_(cs.generate_eight_schools().x))


def test_gibbs_chain_solves_as_a_fixed_point(cuda_device):
    kernel = cs.GibbsKernel(cs.generate_eight_schools(), seed=2, T=512)
    s0 = kernel.initial_state()
    reference = np_(cs.sequential_evaluate(kernel, s0))
    r = cs.run_deer(kernel, s0, cs.DeerConfig(mode="dense", max_iters=200))
    assert r.converged and r.iterations < 100
    assert np.all(np.abs(np_(r.trace) - reference) <= 1e-4 + 1e-3 * np.abs(reference))


@pytest.mark.parametrize("target,eps,L,max_iters", [("rosen", 0.2, 16, None), ("rosen", 0.05, 16, 1),
                                                    ("std", 0.1, 32, None), ("gauss", 0.3, 40, 3)])
def test_batched_inner_solves_match_per_row_runs(cuda_device, target, eps, L, max_iters):
    # cs_leapfrog_batch_solve (one CTA per proposal) against the per-row run_deer
    # loop of samplers.py:301-320 (engine="host"): same states, same fallbacks
    tg = {"rosen": cs.rosenbrock(), "std": cs.std_normal(2),
          "gauss": cs.gaussian(np.zeros(2), np.array([[1.1, 0.0], [0.3, 0.8]]))}[target]
    model = cs.model_logp_grad_hvp(tg)
    kw = {} if max_iters is None else dict(max_iters=max_iters)
    fast = hmc_chain_system(model, eps=eps, L=L, seed=5, T=48, leapfrog_mode="parallel",
                            leapfrog_cfg=cs.DeerConfig(mode="block2x2-stochastic", **kw))
    slow = hmc_chain_system(model, eps=eps, L=L, seed=5, T=48, leapfrog_mode="parallel",
                            leapfrog_cfg=cs.DeerConfig(mode="block2x2-stochastic", engine="host", **kw))
    x0 = np.array([0.5, -0.5])

    def outcome(k):
        try:
            return np_(cs.sequential_evaluate(k, x0)), None
        except ChainDivergedError as e:  # an inner solve tripping its guard propagates, as in the reference
            return None, (e.step, e.iteration)

    (a, ea), (b, eb) = outcome(fast), outcome(slow)
    assert ea == eb
    assert fast.fallback_events == slow.fallback_events
    if ea is not None:
        return
    np.testing.assert_allclose(a, b, atol=1e-10, rtol=1e-10)
    # and one batched step_batch over all rows equals the per-row loop
    S = torch.as_tensor(a, device=cuda_device)
    ts = torch.arange(1, 49, device=cuda_device)
    fast.fallback_events.clear(), slow.fallback_events.clear()
    np.testing.assert_allclose(np_(fast.step_batch(ts, S)), np_(slow.step_batch(ts, S)), atol=1e-10, rtol=1e-10)
    assert fast.fallback_events == slow.fallback_events


def test_parallel_leapfrog_chain_matches_reference_golden(cuda_device):
    # the reference's own HmcKernel(leapfrog_mode="parallel") chain (make_golden.py:
    # Rosenbrock, eps 0.2, L 16, seed 5, T 40), every proposal an inner block
    # quasi-Newton solve -- here all rows' solves batched on the device
    g = np.load(__import__("conftest").GOLDEN + "/hmc_parallel_leapfrog.npz")
    model = cs.model_logp_grad_hvp(cs.rosenbrock(b=0.1, scale2=1.0))
    k = cs.HmcKernel(model, 0.2, 16, seed=5, T=40, leapfrog_mode="parallel",
                     leapfrog_cfg=cs.DeerConfig(mode="block2x2-stochastic"))
    np.testing.assert_allclose(np_(cs.sequential_evaluate(k, np.array([0.5, -0.5]))), g["seq"], atol=1e-8, rtol=1e-8)
    assert [tuple(e) for e in g["fallbacks"]] == [tuple(e) for e in k.fallback_events]


def _wide_gauss(n, seed=0):
    rng = np.random.default_rng(seed)
    Q, _ = np.linalg.qr(rng.normal(size=(n, n)))
    lam = np.exp(rng.uniform(np.log(0.1), np.log(10.0), n))
    return cs.model_logp_grad_hvp(cs.gaussian(np.zeros(n), np.linalg.cholesky((Q * lam) @ Q.T)))


@pytest.mark.parametrize("n,L,eps,T,max_iters", [(16, 24, 0.1, 12, None), (16, 24, 0.1, 6, 2),
                                                 (1000, 100, 0.05, 4, None)])
def test_wide_batched_inner_solves_match_per_row_runs(cuda_device, n, L, eps, T, max_iters):
    # BASELINE cfg 4's proposals (dense Gaussian, n up to 1000, L = 100): every
    # row's inner solve batched (one DMMA GEMM per Newton pass for all rows)
    # against the per-row run_deer loop of samplers.py:301-320 on the streamed
    # engine -- same states, same fallback events
    model = _wide_gauss(n)
    kw = {} if max_iters is None else dict(max_iters=max_iters)
    fast = hmc_chain_system(model, eps=eps, L=L, seed=3, T=T, leapfrog_mode="parallel",
                            leapfrog_cfg=cs.DeerConfig(mode="block2x2-stochastic", **kw))
    slow = hmc_chain_system(model, eps=eps, L=L, seed=3, T=T, leapfrog_mode="parallel",
                            leapfrog_cfg=cs.DeerConfig(mode="block2x2-stochastic", engine="streamed", **kw))
    x0 = np.random.default_rng(1).normal(size=n)
    a = np_(cs.sequential_evaluate(fast, x0))
    b = np_(cs.sequential_evaluate(slow, x0))
    assert fast.fallback_events == slow.fallback_events
    if max_iters is not None:
        assert len(fast.fallback_events) > 0
    np.testing.assert_allclose(a, b, atol=1e-10, rtol=1e-10)

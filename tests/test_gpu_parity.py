"""CUDA path vs the reference (golden fixtures) and the CPU oracle.

Bar (stated here, per north_star): f64 runs match the reference's f64 run_deer
traces to 1e-8 with the SAME Newton iteration count and per-step convergence
record; f32 runs (states/elements in fp32, gate margins in f64) match within
the reference's own convergence envelope |gpu - ref| <= 1e-4 + 1e-3|ref|,
iterations within +-1, identical accept/reject pattern.  Integer/bit work
(counter hash, uniforms, Rademacher probes) is bit-exact.
"""

import numpy as np
import pytest
import torch

import oracle as O
from conftest import golden

pytestmark = pytest.mark.gpu

cs = pytest.importorskip("paper_2508_18413_b200")

F32_ATOL, F32_RTOL = 1e-4, 1e-3


def np_(t):
    return t.detach().cpu().numpy() if torch.is_tensor(t) else np.asarray(t)


def envelope(a, ref, atol=F32_ATOL, rtol=F32_RTOL):
    return bool(np.all(np.abs(np_(a) - ref) <= atol + rtol * np.abs(ref)))


# ---------------------------------------------------------------------------
# noise (noise.py:50-171)


def test_noise_tables_match_reference(cuda_device):
    g = golden("noise")
    layout = {"xi": cs.SlotSpec(3, "standard-normal"), "u": cs.SlotSpec(1, "uniform-0-1"),
              "g": cs.SlotSpec(2, "chi-squared", df=9.1), "g_small": cs.SlotSpec(2, "chi-squared", df=0.1),
              "g_big": cs.SlotSpec(8, "chi-squared", df=20.1)}
    tab = cs.NoiseTable(7, layout, 300)
    np.testing.assert_array_equal(np_(tab.block("u", np.arange(301))), g["u"])          # bit-exact
    np.testing.assert_allclose(np_(tab.block("xi", np.arange(301))), g["xi"], rtol=1e-14, atol=1e-14)
    for k in ("g", "g_small", "g_big"):
        np.testing.assert_allclose(np_(tab.block(k, np.arange(301))), g[k], rtol=1e-11, atol=1e-300)
    big = cs.NoiseTable(2**63 + 12345, {"xi": cs.SlotSpec(2, "standard-normal")}, 10)
    np.testing.assert_allclose(np_(big.block("xi", np.arange(11))), g["xi_bigseed"], rtol=1e-14, atol=1e-14)
    probes = [np_(cs.rademacher_probe(9, it, np.arange(1, 65), k, 6)) for it in range(3) for k in range(3)]
    np.testing.assert_array_equal(np.stack(probes), g["probes"])


def test_chi_squared_inverts_the_gamma_cdf(cuda_device):
    from scipy.special import gammainc

    for df in (0.1, 9.1, 20.1):
        t = cs.NoiseTable(13, {"g": cs.SlotSpec(1, "chi-squared", df=df)}, T=2000)
        u = cs.NoiseTable(13, {"g": cs.SlotSpec(1, "uniform-0-1")}, T=2000)
        x = np_(t.block("g", np.arange(2000)))[:, 0]
        uu = np_(u.block("g", np.arange(2000)))[:, 0]
        assert np.all(x > 0)
        assert np.max(np.abs(gammainc(df / 2.0, x / 2.0) - uu)) < 1e-12   # test_noise.py:72-80


# ---------------------------------------------------------------------------
# scans (pscan.py:273-354)


@pytest.mark.parametrize("T", [1, 257, 1024])
def test_scans_match_reference_golden(cuda_device, T):
    g = golden("scan")
    dev = cuda_device
    t = lambda k: torch.as_tensor(g[k], device=dev)
    out = cs.parallel_affine_solve(cs.DiagElements(t(f"diag_{T}_j"), t(f"diag_{T}_u")), t(f"diag_{T}_s0"))
    np.testing.assert_allclose(np_(out), g[f"diag_{T}_out"], atol=1e-12, rtol=1e-12)
    out = cs.parallel_affine_solve(cs.DenseElements(t(f"dense_{T}_J"), t(f"dense_{T}_u")), t(f"dense_{T}_s0"))
    np.testing.assert_allclose(np_(out), g[f"dense_{T}_out"], atol=1e-12, rtol=1e-12)
    el = cs.Block2x2Elements(*(t(f"block_{T}_{k}") for k in "abcdu"))
    out = cs.parallel_affine_solve(el, t(f"block_{T}_s0"))
    np.testing.assert_allclose(np_(out), g[f"block_{T}_out"], atol=1e-12, rtol=1e-12)


def test_scan_kats(cuda_device):
    e = cs.DiagElements(torch.tensor([[2.0], [3.0], [4.0]], device=cuda_device),
                        torch.ones((3, 1), dtype=torch.float64, device=cuda_device))
    np.testing.assert_array_equal(np_(cs.parallel_affine_solve(e, torch.tensor([1.0], device=cuda_device)))[:, 0],
                                  [3.0, 10.0, 41.0])
    T, D = 64, 3
    e = cs.DiagElements(torch.ones((T, D), dtype=torch.float64, device=cuda_device),
                        torch.zeros((T, D), dtype=torch.float64, device=cuda_device))
    s0 = torch.tensor([4.0, -1.0, 0.25], dtype=torch.float64, device=cuda_device)
    assert bool((cs.parallel_affine_solve(e, s0) == s0).all())


@pytest.mark.parametrize("D", [1, 2, 5, 18, 64, 65, 100, 300])
@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_diag_and_block_scans_vs_oracle(cuda_device, D, dtype):
    rng = np.random.default_rng(D)
    T = 20_011
    j = rng.uniform(-0.95, 0.95, (T, D))
    u = rng.normal(size=(T, D))
    s0 = rng.normal(size=D)
    want = O.parallel_affine_solve(O.DiagElements(j, u), s0, workers=8)
    tt = lambda x: torch.as_tensor(x, dtype=dtype, device=cuda_device)
    got = np_(cs.parallel_affine_solve(cs.DiagElements(tt(j), tt(u)), tt(s0)))
    tol = 1e-11 if dtype == torch.float64 else 2e-5
    np.testing.assert_allclose(got, want, atol=tol * 10, rtol=tol)
    a, b, c, d = (rng.uniform(-0.65, 0.65, (T, D)) for _ in range(4))
    ub = rng.normal(size=(T, 2 * D))
    s0b = rng.normal(size=2 * D)
    want = O.parallel_affine_solve(O.Block2x2Elements(a, b, c, d, ub), s0b, workers=8)
    got = np_(cs.parallel_affine_solve(cs.Block2x2Elements(tt(a), tt(b), tt(c), tt(d), tt(ub)), tt(s0b)))
    np.testing.assert_allclose(got, want, atol=tol * 10, rtol=tol)


@pytest.mark.parametrize("D", [1, 2, 3, 4, 6, 8])
def test_dense_scan_vs_oracle(cuda_device, D):
    rng = np.random.default_rng(40 + D)
    T = 5003
    J = rng.normal(size=(T, D, D))
    J *= (0.9 / np.abs(np.linalg.eigvals(J)).max(axis=-1))[:, None, None]
    u = rng.normal(size=(T, D))
    s0 = rng.normal(size=D)
    want = O.parallel_affine_solve(O.DenseElements(J, u), s0, workers=8)
    tt = lambda x: torch.as_tensor(x, device=cuda_device)
    got = np_(cs.parallel_affine_solve(cs.DenseElements(tt(J), tt(u)), tt(s0)))
    np.testing.assert_allclose(got, want, atol=1e-10, rtol=1e-10)


@pytest.mark.parametrize("D,T", [(9, 1), (9, 3001), (16, 2000), (33, 777), (100, 1), (100, 2049), (128, 1500),
                                 (64, 5001), (100, 20001)])
@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_wide_dense_scan_vs_oracle(cuda_device, D, T, dtype):
    # chunked reduce / carry / replay for 8 < D <= 128 (cs_dense.cu; A12 at cfg 3's D = 100);
    # f32 with D % 4 == 0, D < 128: chunk aggregates by the tree-ordered tcgen05
    # composition (odd tails at several levels for T = 5001, 20001)
    rng = np.random.default_rng(7 * D + T)
    J = rng.normal(size=(T, D, D)) * (0.9 / (2.0 * np.sqrt(D)))  # spectral radius ~0.45
    u = rng.normal(size=(T, D))
    s0 = rng.normal(size=D)
    tt = lambda x: torch.as_tensor(x, dtype=dtype, device=cuda_device)
    Jd, ud, s0d = (np_(tt(x)).astype(np.float64) for x in (J, u, s0))  # the inputs the kernel sees
    want = O.parallel_affine_solve(O.DenseElements(Jd, ud), s0d, workers=8)
    got = np_(cs.parallel_affine_solve(cs.DenseElements(tt(J), tt(u)), tt(s0)))
    tol = 1e-10 if dtype == torch.float64 else 2e-5
    np.testing.assert_allclose(got, want, atol=tol * 10, rtol=tol)


def test_wide_dense_scan_kat_and_errors(cuda_device):
    # J = 0.5 I for every step: s_t = 0.5 s_{t-1} + 1 -> 2 - 2^-t (s0 = 1 gives 2 - 2^-t)
    T, D = 700, 40
    J = torch.eye(D, dtype=torch.float64, device=cuda_device).expand(T, D, D).contiguous() * 0.5
    u = torch.ones((T, D), dtype=torch.float64, device=cuda_device)
    got = np_(cs.parallel_affine_solve(cs.DenseElements(J, u), torch.ones(D, dtype=torch.float64, device=cuda_device)))
    want = 2.0 - 0.5 ** np.arange(1, T + 1)
    np.testing.assert_allclose(got, np.repeat(want[:, None], D, axis=1), rtol=1e-13, atol=1e-13)
    with pytest.raises(cs.StructuralError):
        cs.parallel_affine_solve(cs.DenseElements(J, u), torch.ones(D + 1, dtype=torch.float64, device=cuda_device))


@pytest.mark.parametrize("D,T", [(129, 1), (129, 1201), (200, 300), (257, 150)])
@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_xl_dense_scan_vs_oracle(cuda_device, D, T, dtype):
    # D > 128 (cs_dense_xl.cu): batched-GEMM chunk maps, f64 carry, CTA-per-chunk
    # replay; partial last chunks at T = 1201 (c = 9) and T = 150 (c = 8)
    rng = np.random.default_rng(3 * D + T)
    J = rng.normal(size=(T, D, D)) * (0.9 / (2.0 * np.sqrt(D)))
    u = rng.normal(size=(T, D))
    s0 = rng.normal(size=D)
    tt = lambda x: torch.as_tensor(x, dtype=dtype, device=cuda_device)
    Jd, ud, s0d = (np_(tt(x)).astype(np.float64) for x in (J, u, s0))
    want = O.parallel_affine_solve(O.DenseElements(Jd, ud), s0d, workers=8)
    got = np_(cs.parallel_affine_solve(cs.DenseElements(tt(J), tt(u)), tt(s0)))
    tol = 1e-10 if dtype == torch.float64 else 2e-5
    np.testing.assert_allclose(got, want, atol=tol * 10, rtol=tol)


def test_xl_dense_scan_kat(cuda_device):
    T, D = 333, 150
    J = torch.eye(D, dtype=torch.float64, device=cuda_device).expand(T, D, D).contiguous() * 0.5
    u = torch.ones((T, D), dtype=torch.float64, device=cuda_device)
    got = np_(cs.parallel_affine_solve(cs.DenseElements(J, u), torch.ones(D, dtype=torch.float64, device=cuda_device)))
    want = 2.0 - 0.5 ** np.arange(1, T + 1)
    np.testing.assert_allclose(got, np.repeat(want[:, None], D, axis=1), rtol=1e-13, atol=1e-13)


# ---------------------------------------------------------------------------
# systems: batched f_t and JVPs vs the oracle (samplers.py)


def _pair(kind, dtype=torch.float64, T=64):
    if kind == "mala_gauss":
        mu, L = [1.0, -1.0], [[1.0, 0.0], [-0.6, 1.2]]
        return (cs.MalaKernel(cs.model_logp_grad_hvp(cs.gaussian(mu, L)), 0.4, seed=3, T=T, dtype=dtype),
                O.MalaKernel(O.gaussian(mu, L), 0.4, seed=3, T=T))
    if kind == "mala_mog":
        return (cs.MalaKernel(cs.model_logp_grad_hvp(cs.mog()), 0.1, seed=5, T=T, dtype=dtype),
                O.MalaKernel(O.mog(), 0.1, seed=5, T=T))
    if kind == "mala_std5":
        return (cs.MalaKernel(cs.model_logp_grad_hvp(cs.std_normal(5)), 0.3, seed=1, T=T, dtype=dtype),
                O.MalaKernel(O.std_normal(5), 0.3, seed=1, T=T))
    if kind == "hmc_rosen":
        return (cs.HmcKernel(cs.model_logp_grad_hvp(cs.rosenbrock(b=0.1, scale2=1.0)), 0.5, 8, seed=0, T=T,
                             dtype=dtype),
                O.HmcKernel(O.rosenbrock(b=0.1, scale2=1.0), 0.5, 8, seed=0, T=T))
    if kind == "hmc_gauss_mass":
        mu, L = [0.5, 0.0, -0.5], [[1.0, 0, 0], [0.3, 1.1, 0], [0.0, -0.2, 0.9]]
        return (cs.HmcKernel(cs.model_logp_grad_hvp(cs.gaussian(mu, L)), 0.2, 5, seed=2, T=T,
                             mass=[1.0, 2.0, 0.5], dtype=dtype),
                O.HmcKernel(O.gaussian(mu, L), 0.2, 5, seed=2, T=T, mass=[1.0, 2.0, 0.5]))
    if kind == "leapfrog_rosen":
        return (cs.LeapfrogSystem(cs.model_logp_grad_hvp(cs.rosenbrock()), 0.05, 16, probe_seed=4, dtype=dtype),
                O.LeapfrogSystem(O.rosenbrock(), 0.05, 16, probe_seed=4))
    if kind == "gibbs":
        data_c = cs.generate_eight_schools()
        data_o = O.generate_eight_schools()
        return cs.GibbsKernel(data_c, seed=0, T=T, dtype=dtype), O.GibbsKernel(data_o, seed=0, T=T)
    raise KeyError(kind)


SYSTEMS = ["mala_gauss", "mala_mog", "mala_std5", "hmc_rosen", "hmc_gauss_mass", "leapfrog_rosen", "gibbs"]


@pytest.mark.parametrize("kind", SYSTEMS)
def test_system_step_and_jvp_vs_oracle(cuda_device, kind):
    gs, os_ = _pair(kind)
    rng = np.random.default_rng(11)
    n = os_.T if kind != "leapfrog_rosen" else 16
    D = os_.dim
    S = rng.normal(size=(n, D)) * 0.7
    if kind == "gibbs":
        S[:, 0] = np.abs(S[:, 0]) + 1.0
        S[:, 10:] = np.abs(S[:, 10:]) * 50 + 1.0
    V = rng.normal(size=(n, D))
    ts = np.arange(1, n + 1)
    np.testing.assert_allclose(np_(gs.step_batch(ts, S)), os_.step_batch(ts, S), rtol=1e-11, atol=1e-11)
    np.testing.assert_allclose(np_(gs.jvp_batch(ts, S, V)), os_.jvp_batch(ts, S, V), rtol=1e-9, atol=1e-9)
    if hasattr(os_, "relaxed_jvp_batch"):
        np.testing.assert_allclose(np_(gs.relaxed_jvp_batch(ts, S, V)), os_.relaxed_jvp_batch(ts, S, V),
                                   rtol=1e-9, atol=1e-9)
    if kind == "leapfrog_rosen":
        for it in (0, 3):
            got = gs.block_jacobian_batch(ts, S, 2, it)
            want = os_.block_jacobian_batch(ts, S, 2, it)
            for g_, w_ in zip(got, want):
                np.testing.assert_allclose(np_(g_), w_, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("kind", ["mala_gauss", "mala_mog", "hmc_rosen", "gibbs", "leapfrog_rosen"])
def test_sequential_evaluate_vs_oracle(cuda_device, kind):
    gs, os_ = _pair(kind, T=500)
    if kind == "gibbs":
        s0 = os_.initial_state()
        np.testing.assert_allclose(np_(gs.initial_state()), s0, rtol=1e-11)
    elif kind == "leapfrog_rosen":
        s0 = np.array([0.4, -0.3, 0.6, 0.1])
    else:
        s0 = np.zeros(os_.dim)
    T = os_.T
    want = O.sequential_evaluate(os_, s0, T)
    got = np_(cs.sequential_evaluate(gs, s0, T))
    np.testing.assert_allclose(got, want, rtol=1e-9, atol=1e-9)


# ---------------------------------------------------------------------------
# whole-chain solves vs the reference's own run_deer (golden)


def _deer_cmp(res, g, prefix, dtype, exact_iters=True):
    it_ref = int(g[prefix + "iterations"])
    if dtype == torch.float64:
        assert res.iterations == it_ref
        np.testing.assert_allclose(np_(res.trace), g[prefix + "trace"], atol=1e-8, rtol=1e-8)
        np.testing.assert_array_equal(np_(res.per_step_converged_at), g[prefix + "psca"])
        np.testing.assert_allclose(res.delta_history, g[prefix + "delta_history"], rtol=1e-6, atol=1e-12)
    else:
        assert abs(res.iterations - it_ref) <= 1
        assert envelope(res.trace, g[prefix + "trace"])
    assert res.converged == bool(g[prefix + "converged"])


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_run_deer_mala_gauss2d(cuda_device, dtype):
    g = golden("mala_gauss2d")
    m = cs.model_logp_grad_hvp(cs.gaussian([1.0, -1.0], [[1.0, 0.0], [-0.6, 1.2]]))
    k = cs.MalaKernel(m, 0.4, seed=0, T=2000, dtype=dtype)
    np.testing.assert_allclose(np_(cs.sequential_evaluate(k, np.zeros(2))), g["seq"], atol=1e-6 if dtype == torch.float32 else 1e-10)
    r = cs.run_deer(k, np.zeros(2), cs.DeerConfig(mode="dense"))
    assert r.stats["path"] == "fused"
    _deer_cmp(r, g, "dense_", dtype)
    _deer_cmp(cs.run_deer(k, np.zeros(2), cs.DeerConfig(mode="diag-stochastic")), g, "diag_", dtype)
    _deer_cmp(cs.run_deer(k, np.zeros(2), cs.DeerConfig(mode="dense", atol=1e-6, rtol=1e-5)), g, "tight_", dtype)


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_run_deer_mala_rosen2d(cuda_device, dtype):
    g = golden("mala_rosen2d")
    k = cs.MalaKernel(cs.model_logp_grad_hvp(cs.rosenbrock(b=0.1, scale2=1.0)), 0.5, seed=0, T=2000, dtype=dtype)
    _deer_cmp(cs.run_deer(k, np.zeros(2), cs.DeerConfig(mode="dense")), g, "dense_", dtype)


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_run_deer_hmc_rosen2d(cuda_device, dtype):
    g = golden("hmc_rosen2d")
    m = cs.model_logp_grad_hvp(cs.rosenbrock(a=0.0, b=0.1, scale1=1.0, scale2=1.0))
    k = cs.HmcKernel(m, 0.5, 8, seed=0, T=5000, dtype=dtype)
    np.testing.assert_allclose(np_(cs.sequential_evaluate(k, np.zeros(2))), g["seq"],
                               atol=1e-5 if dtype == torch.float32 else 1e-9)
    _deer_cmp(cs.run_deer(k, np.zeros(2), cs.DeerConfig(mode="diag-stochastic", clip=1.0)), g, "diagclip_", dtype)
    _deer_cmp(cs.run_deer(k, np.zeros(2), cs.DeerConfig(mode="dense", damping=0.5, clip=1.0, atol=1e-6, rtol=1e-5)),
              g, "dense_", dtype)


def test_run_deer_mog_damped(cuda_device):
    g = golden("mala_mog2d")
    k = cs.MalaKernel(cs.model_logp_grad_hvp(cs.mog()), 0.1, seed=3, T=1000)
    _deer_cmp(cs.run_deer(k, np.zeros(2), cs.DeerConfig(mode="diag-stochastic", damping=0.5, max_iters=300)),
              g, "damped_", torch.float64)


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_run_deer_gibbs(cuda_device, dtype):
    g = golden("gibbs_schools")
    k = cs.GibbsKernel(cs.generate_eight_schools(), seed=0, T=3000, dtype=dtype)
    s0 = k.initial_state()
    np.testing.assert_allclose(np_(s0), g["s0"], rtol=1e-10 if dtype == torch.float64 else 1e-6)
    cfg = cs.DeerConfig(mode="diag-stochastic", hutchinson_samples=3, preconditioner=k.recommended_preconditioner(),
                        max_iters=400)
    r = cs.run_deer(k, g["s0"], cfg)
    _deer_cmp(r, g, "diag3_", dtype)


@pytest.mark.parametrize("mode,kw", [("diag-stochastic", dict(clip=1.0)), ("dense", dict(damping=0.5, clip=1.0))])
def test_engines_agree(cuda_device, mode, kw):
    m = cs.model_logp_grad_hvp(cs.rosenbrock(a=0.0, b=0.1, scale1=1.0, scale2=1.0))
    k = cs.HmcKernel(m, 0.5, 8, seed=0, T=3000)
    runs = {e: cs.run_deer(k, np.zeros(2), cs.DeerConfig(mode=mode, engine=e, **kw))
            for e in ("fused", "streamed", "host")}
    for e, r in runs.items():
        assert r.stats["path"] == e
    a = runs["fused"]
    for e in ("streamed", "host"):
        b = runs[e]
        assert a.iterations == b.iterations and a.converged == b.converged
        np.testing.assert_allclose(np_(a.trace), np_(b.trace), atol=1e-10)
        np.testing.assert_array_equal(np_(a.per_step_converged_at), np_(b.per_step_converged_at))
        np.testing.assert_allclose(a.delta_history, b.delta_history, rtol=1e-9, atol=1e-15)


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_streamed_engine_golden(cuda_device, dtype):
    g = golden("gibbs_schools")
    k = cs.GibbsKernel(cs.generate_eight_schools(), seed=0, T=3000, dtype=dtype)
    cfg = cs.DeerConfig(mode="diag-stochastic", hutchinson_samples=3, preconditioner=k.recommended_preconditioner(),
                        max_iters=400, engine="streamed")
    r = cs.run_deer(k, g["s0"], cfg)
    assert r.stats["path"] == "streamed"
    _deer_cmp(r, g, "diag3_", dtype)
    g = golden("hmc_rosen2d")
    m = cs.model_logp_grad_hvp(cs.rosenbrock(a=0.0, b=0.1, scale1=1.0, scale2=1.0))
    k = cs.HmcKernel(m, 0.5, 8, seed=0, T=5000, dtype=dtype)
    _deer_cmp(cs.run_deer(k, np.zeros(2), cs.DeerConfig(mode="diag-stochastic", clip=1.0, engine="streamed")),
              g, "diagclip_", dtype)
    _deer_cmp(cs.run_deer(k, np.zeros(2), cs.DeerConfig(mode="dense", damping=0.5, clip=1.0, atol=1e-6, rtol=1e-5,
                                                        engine="streamed")), g, "dense_", dtype)
    # leapfrog block elements through the streamed engine (test_deer.py:250-261 one-shot)
    lf = cs.LeapfrogSystem(cs.model_logp_grad_hvp(cs.std_normal(2)), 0.1, 64, dtype=dtype)
    r = cs.run_deer(lf, np.array([1.0, -0.5, 0.3, 0.8]), cs.DeerConfig(mode="block2x2-stochastic", engine="streamed"))
    assert r.stats["path"] == "streamed" and r.converged and r.iterations == 1


def test_run_deer_leapfrog_block_and_window(cuda_device):
    g = golden("mala_window")
    k = cs.MalaKernel(cs.model_logp_grad_hvp(cs.std_normal(2)), 0.3, seed=6, T=512)
    r = cs.run_deer(k, np.array([1.0, 0.0]), cs.DeerConfig(mode="dense", window_len=64, max_iters=2000))
    assert r.stats["path"] == "streamed-window"  # the window runs on the device engine
    _deer_cmp(r, g, "win64_", torch.float64)
    k1 = cs.MalaKernel(cs.model_logp_grad_hvp(cs.std_normal(2)), 0.3, seed=6, T=40)
    r = cs.run_deer(k1, np.array([1.0, 0.0]), cs.DeerConfig(mode="dense", window_len=1, max_iters=500))
    assert r.stats["path"] == "streamed-window"
    _deer_cmp(r, g, "win1_", torch.float64)
    # and the host engine's window loop agrees on both
    for kk, cfg, pre in ((k, cs.DeerConfig(mode="dense", window_len=64, max_iters=2000, engine="host"), "win64_"),
                         (k1, cs.DeerConfig(mode="dense", window_len=1, max_iters=500, engine="host"), "win1_")):
        h = cs.run_deer(kk, np.array([1.0, 0.0]), cfg)
        assert h.stats["path"] == "host"
        _deer_cmp(h, g, pre, torch.float64)
    # block one-shot on a Gaussian leapfrog (test_deer.py:250-261)
    lf = cs.LeapfrogSystem(cs.model_logp_grad_hvp(cs.std_normal(2)), 0.1, 64)
    s0 = np.array([1.0, -0.5, 0.3, 0.8])
    r = cs.run_deer(lf, s0, cs.DeerConfig(mode="block2x2-stochastic"))
    assert r.converged and r.iterations == 1
    np.testing.assert_allclose(np_(r.trace), np_(cs.sequential_evaluate(lf, s0)), atol=1e-9)


# ---------------------------------------------------------------------------
# GEMM-evaluated systems: logistic-regression MALA (cfg 3) and the wide
# Gaussian leapfrog (cfg 4)


def test_synthetic_credit_like_matches_reference(cuda_device):
    g = golden("mala_blr100")
    X, y, beta = cs.synthetic_credit_like(seed=20250819, n=1000, dim=100)
    np.testing.assert_allclose(X, g["X"], rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(beta, g["beta_star"], rtol=1e-13, atol=1e-13)
    np.testing.assert_array_equal(y, g["y"])


def test_run_deer_blr_gemm_path(cuda_device):
    g = golden("mala_blr100")
    m = cs.model_logp_grad_hvp(cs.blr(g["X"], g["y"], 1.0))
    k = cs.MalaKernel(m, 0.003, seed=4, T=300)
    assert not k.kernels
    np.testing.assert_allclose(np_(cs.sequential_evaluate(k, np.zeros(100))), g["seq"], atol=1e-9, rtol=1e-9)
    # GEMM-backed element builder on the streamed engine (cs_blr.cu) and the
    # host engine's torch evaluation: both must reproduce the reference run
    r = cs.run_deer(k, np.zeros(100), cs.DeerConfig(mode="diag-stochastic"))
    assert r.stats["path"] == "streamed"
    _deer_cmp(r, g, "diag_", torch.float64)
    h = cs.run_deer(k, np.zeros(100), cs.DeerConfig(mode="diag-stochastic", engine="host"))
    assert h.stats["path"] == "host"
    _deer_cmp(h, g, "diag_", torch.float64)


@pytest.mark.parametrize("N,D,T", [(1000, 100, 37), (77, 9, 5), (512, 128, 3), (33, 64, 300), (1000, 100, 1000)])
@pytest.mark.parametrize("hook", ["cs_debug_gram", "cs_debug_pair_gram"])
def test_tcgen05_weighted_gram(cuda_device, N, D, T, hook):
    # the 5th-gen tensor-core (tcgen05/TMEM) Hessian term X^T diag(w_t) X against
    # an f64 evaluation -- per step (cs_debug_gram) and as one pair-Gram GEMM over
    # all steps (cs_debug_pair_gram); TF32 operands -> relative error ~1e-3 of the
    # term scale
    from paper_2508_18413_b200 import _lib

    g = torch.Generator(device=cuda_device).manual_seed(N + D)
    X = torch.randn((N, D), generator=g, device=cuda_device, dtype=torch.float64)
    W = torch.rand((T, N), generator=g, device=cuda_device, dtype=torch.float64) * 0.25
    H = torch.empty((T, 128, 128), device=cuda_device, dtype=torch.float32)
    _lib.check(getattr(_lib.load(), hook)(_lib.ptr(X), N, D, _lib.ptr(W), T, _lib.ptr(H), _lib.stream_ptr()))
    torch.cuda.synchronize()
    want = torch.einsum("nd,tn,ne->tde", X, W, X)
    got = H[:, :D, :D].double()
    scale = torch.einsum("nd,tn,ne->tde", X.abs(), W, X.abs())
    assert float(((got - want).abs() / (scale + 1e-30)).max()) < 4e-3
    assert torch.count_nonzero(H[:, D:, :]) == 0 and torch.count_nonzero(H[:, :, D:]) == 0
    assert torch.equal(H, H.transpose(1, 2))


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_run_deer_blr_dense_wide(cuda_device, dtype):
    # cfg3 "full vs diagonal": dense Newton at D = 100 -- Jacobians from the
    # system's jvps, the wide dense scan (cs_dense.cu) -- against the reference
    g0, g = golden("mala_blr100"), golden("mala_blr100_dense")
    m = cs.model_logp_grad_hvp(cs.blr(g0["X"], g0["y"], 1.0))
    k = cs.MalaKernel(m, 0.003, seed=4, T=300, dtype=dtype)
    # closed-form element builder on the streamed engine (cs_blr.cu, k_bd_final)
    r = cs.run_deer(k, np.zeros(100), cs.DeerConfig(mode="dense"))
    assert r.stats["path"] == "streamed"
    _deer_cmp(r, g, "dense_", dtype)
    # and the reference's own construction: J column by column from D jvps (host engine)
    h = cs.run_deer(k, np.zeros(100), cs.DeerConfig(mode="dense", engine="host"))
    assert h.stats["path"] == "host"
    _deer_cmp(h, g, "dense_", dtype)


@pytest.mark.parametrize("mode", ["dense", "diag-stochastic"])
def test_blr_concurrent_streams_match_serial(cuda_device, mode):
    # the logistic-regression builders share per-device scratch: solves from two
    # threads on two streams must see it handed off in stream order (no
    # overwrite mid-flight) and reproduce the serial traces bit for bit
    import threading

    g0 = golden("mala_blr100")
    m = cs.model_logp_grad_hvp(cs.blr(g0["X"], g0["y"], 1.0))

    def solve(seed):
        k = cs.MalaKernel(m, 0.003, seed=seed, T=400, dtype=torch.float32)
        return cs.run_deer(k, np.zeros(100), cs.DeerConfig(mode=mode, max_iters=30))

    want = {sd: solve(sd).trace.cpu() for sd in (4, 5)}
    out, errs = {}, []

    def worker(sd):
        try:
            s = torch.cuda.Stream(device=cuda_device)
            with torch.cuda.stream(s):
                for _ in range(3):
                    r = solve(sd)
                    out.setdefault(sd, []).append(r.trace.cpu())
        except Exception as e:  # surfaced below
            errs.append(e)

    ths = [threading.Thread(target=worker, args=(sd,)) for sd in (4, 5)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    assert not errs, errs
    for sd in (4, 5):
        assert all(torch.equal(x, want[sd]) for x in out[sd])


@pytest.mark.parametrize("kw", [dict(damping=0.7), dict(preconditioner="ramp"), dict(clip=0.5),
                                dict(damping=0.8, preconditioner="ramp", clip=2.0)])
def test_blr_dense_builder_options_match_host_engine(cuda_device, kw):
    # the closed-form element (u from J prev in closed form when unclipped) against
    # the host engine's jvp-built J + elementwise formation, with preconditioner /
    # damping / clip (deer.py:161-170)
    g0 = golden("mala_blr100")
    kw = dict(kw)
    if kw.get("preconditioner") == "ramp":
        kw["preconditioner"] = np.linspace(0.5, 2.0, 100)
    m = cs.model_logp_grad_hvp(cs.blr(g0["X"], g0["y"], 1.0))
    k = cs.MalaKernel(m, 0.003, seed=4, T=150)
    cfg = cs.DeerConfig(mode="dense", max_iters=60, **kw)
    r = cs.run_deer(k, np.zeros(100), cfg)
    h = cs.run_deer(k, np.zeros(100), cs.DeerConfig(mode="dense", max_iters=60, engine="host", **kw))
    assert r.stats["path"] == "streamed" and h.stats["path"] == "host"
    assert r.iterations == h.iterations and r.converged == h.converged
    np.testing.assert_allclose(np_(r.trace), np_(h.trace), atol=1e-9, rtol=1e-9)
    np.testing.assert_array_equal(np_(r.per_step_converged_at), np_(h.per_step_converged_at))


@pytest.mark.parametrize("D", [9, 100, 128])
def test_blr_dense_f32_builder_widths(cuda_device, D):
    # the f32 dense builder (pair-Gram tcgen05 Hessian + element kernel: scalar J
    # rows at D % 4 != 0, 16-byte rows otherwise, DP = 112 / 128 tiles) converges
    # to the sequential chain, like the host engine's jvp-built Jacobians
    X, y, _ = cs.synthetic_credit_like(seed=7 + D, n=400, dim=D)
    m = cs.model_logp_grad_hvp(cs.blr(X, y, 1.0))
    k = cs.MalaKernel(m, 0.002, seed=3, T=257, dtype=torch.float32)
    seq = np_(cs.sequential_evaluate(k, np.zeros(D)))
    r = cs.run_deer(k, np.zeros(D), cs.DeerConfig(mode="dense", atol=1e-6, rtol=1e-5, max_iters=120))
    h = cs.run_deer(k, np.zeros(D), cs.DeerConfig(mode="dense", atol=1e-6, rtol=1e-5, max_iters=120, engine="host"))
    assert r.stats["path"] == "streamed" and h.stats["path"] == "host"
    assert r.converged and h.converged
    assert abs(r.iterations - h.iterations) <= 3
    np.testing.assert_allclose(np_(r.trace), seq, atol=2e-4, rtol=2e-4)
    np.testing.assert_allclose(np_(h.trace), seq, atol=2e-4, rtol=2e-4)


def test_run_deer_leapfrog_gauss200(cuda_device):
    g = golden("leapfrog_gauss200")
    m = cs.model_logp_grad_hvp(cs.gaussian(np.zeros(200), g["chol"]))
    lf = cs.LeapfrogSystem(m, 0.05, 100, probe_seed=0)
    assert not lf.kernels
    np.testing.assert_allclose(np_(cs.sequential_evaluate(lf, g["s0"])), g["seq"], atol=1e-9, rtol=1e-9)
    _deer_cmp(cs.run_deer(lf, g["s0"], cs.DeerConfig(mode="block2x2-stochastic")), g, "block_", torch.float64)
    _deer_cmp(cs.run_deer(lf, g["s0"], cs.DeerConfig(mode="diag-stochastic")), g, "diag_", torch.float64)


def test_wide_leapfrog_builder_matches_host_engine(cuda_device):
    # the GEMM-backed element builder (cuBLAS DGEMM + fused epilogue) against the
    # host engine's torch evaluation of the same LeapfrogSystem (samplers.py:165-222)
    g = golden("leapfrog_gauss200")
    m = cs.model_logp_grad_hvp(cs.gaussian(np.zeros(200), g["chol"]))
    for dt, tol in ((torch.float64, 1e-10), (torch.float32, 2e-4)):
        lf = cs.LeapfrogSystem(m, 0.05, 100, probe_seed=0, dtype=dt)
        cfg = dict(mode="block2x2-stochastic", damping=0.9)
        a = cs.run_deer(lf, g["s0"], cs.DeerConfig(engine="streamed", **cfg))
        b = cs.run_deer(lf, g["s0"], cs.DeerConfig(engine="host", **cfg))
        assert a.stats["path"] == "streamed" and b.stats["path"] == "host"
        assert abs(a.iterations - b.iterations) <= (0 if dt == torch.float64 else 1)
        np.testing.assert_allclose(np_(a.trace), np_(b.trace), atol=tol, rtol=tol)


def _cfg4_gaussian(D=1000):
    rng = np.random.default_rng(0)
    Q, _ = np.linalg.qr(rng.normal(size=(D, D)))
    lam = np.exp(rng.uniform(np.log(0.1), np.log(10.0), D))
    P = (Q * lam) @ Q.T
    return np.linalg.cholesky(P)


def test_leapfrog_block_cfg4_full_size_vs_oracle(cuda_device):
    # BASELINE cfg 4: HMC proposal of L=100 leapfrog steps, Gaussian D=1000, block quasi-Newton
    D, eps, L = 1000, 0.05, 100
    Lc = _cfg4_gaussian(D)
    om = O.gaussian(np.zeros(D), Lc)
    x0 = np.random.default_rng(1).normal(size=D)
    v0 = np.random.default_rng(2).normal(size=D)
    s0 = np.concatenate([x0, v0 + 0.5 * eps * om.grad(x0)])
    ref = O.run_deer(O.LeapfrogSystem(om, eps, L, probe_seed=0), s0, O.DeerConfig(mode="block2x2-stochastic"))
    lf = cs.LeapfrogSystem(cs.model_logp_grad_hvp(cs.gaussian(np.zeros(D), Lc)), eps, L, probe_seed=0)
    r = cs.run_deer(lf, s0, cs.DeerConfig(mode="block2x2-stochastic"))
    assert r.iterations == ref.iterations
    np.testing.assert_allclose(np_(r.trace), ref.trace, atol=1e-8, rtol=1e-8)
    np.testing.assert_array_equal(np_(r.per_step_converged_at), ref.per_step_converged_at)


# ---------------------------------------------------------------------------
# the sharded driver's CUDA shard ops (world size 1 here; the multi-rank
# exchange is covered with gloo in test_sharded_gloo.py)


@pytest.mark.parametrize("mode,kw", [("diag-stochastic", dict(clip=1.0)), ("dense", dict(damping=0.5, clip=1.0))])
def test_sharded_driver_cuda_ops_single_rank(cuda_device, mode, kw):
    from paper_2508_18413_b200.sharded import run_deer_sharded

    m = cs.model_logp_grad_hvp(cs.rosenbrock(a=0.0, b=0.1, scale1=1.0, scale2=1.0))
    k = cs.HmcKernel(m, 0.5, 8, seed=0, T=3000)
    ref = cs.run_deer(k, np.zeros(2), cs.DeerConfig(mode=mode, **kw))
    r = run_deer_sharded(k, np.zeros(2), cs.DeerConfig(mode=mode, **kw))
    assert r.iterations == ref.iterations and r.converged == ref.converged
    np.testing.assert_allclose(np_(r.trace), np_(ref.trace), atol=1e-10)
    np.testing.assert_array_equal(np_(r.per_step_converged_at), np_(ref.per_step_converged_at))


@pytest.mark.parametrize("which,mode", [("mala", "diag-stochastic"), ("mala", "dense"), ("hmc", "diag-stochastic"),
                                        ("gibbs", "diag-stochastic"), ("leapfrog", "block2x2-stochastic")])
def test_elements_range_equals_whole_chain_rows(cuda_device, which, mode):
    # cs_system_elements_range (one rank's T shard): noise and probes at the
    # absolute step, the halo row as the state before the shard -> bit-identical
    # to rows lo..hi-1 of the whole chain's elements
    import ctypes

    from paper_2508_18413_b200 import _lib
    from paper_2508_18413_b200.deer import _MODE_CODE, _STATS_BYTES, _parse_stats

    if which == "mala":
        k = cs.MalaKernel(cs.model_logp_grad_hvp(cs.gaussian([1.0, -1.0], [[1.0, 0.0], [-0.6, 1.2]])), 0.4, seed=3, T=5000)
        s0 = torch.zeros(2, dtype=torch.float64, device=cuda_device)
    elif which == "hmc":
        k = cs.HmcKernel(cs.model_logp_grad_hvp(cs.rosenbrock(a=0.0, b=0.1, scale1=1.0, scale2=1.0)), 0.5, 8, seed=1, T=5000)
        s0 = torch.zeros(2, dtype=torch.float64, device=cuda_device)
    elif which == "gibbs":
        k = cs.GibbsKernel(cs.generate_eight_schools(), seed=2, T=5000)
        s0 = torch.as_tensor(k.initial_state(), device=cuda_device)
    else:
        k = cs.LeapfrogSystem(cs.model_logp_grad_hvp(cs.rosenbrock(b=0.1, scale2=1.0)), 0.1, 64, probe_seed=4)
        s0 = torch.tensor([0.3, -0.2, 1.0, 0.5], dtype=torch.float64, device=cuda_device)
    T, D = k.T, k.dim
    guess = cs.sequential_evaluate(k, s0).contiguous()
    lib = _lib.load()
    d = k.desc()
    c = _lib.cs_deer_config()
    c.mode = _MODE_CODE[mode]
    c.atol, c.rtol, c.max_iters, c.hutchinson_samples = 1e-4, 1e-3, 100, 3 if which == "gibbs" else 1
    c.damping, c.clip, c.preconditioner = 1.0, float("inf"), 0
    half = D // 2 if mode == "block2x2-stochastic" else D

    def build(t0, n, prev, g):
        if mode == "diag-stochastic":
            E = [torch.empty((n, D), dtype=torch.float64, device=cuda_device)]
        elif mode == "dense":
            E = [torch.empty((n, D, D), dtype=torch.float64, device=cuda_device)]
        else:
            E = [torch.empty((n, half), dtype=torch.float64, device=cuda_device) for _ in range(4)]
        u = torch.empty((n, D), dtype=torch.float64, device=cuda_device)
        st = torch.zeros(_STATS_BYTES, dtype=torch.uint8, device=cuda_device)
        ptrs = [_lib.ptr(x) for x in E] + [_lib.ptr(None)] * (4 - len(E))
        rc = lib.cs_system_elements_range(ctypes.byref(d), ctypes.byref(c), _lib.dtype_code(torch.float64), 2, t0, n,
                                          _lib.ptr(prev.contiguous()), _lib.ptr(g.contiguous()), *ptrs, _lib.ptr(u),
                                          _lib.ptr(st), _lib.stream_ptr())
        _lib.check(rc)
        return [np_(x) for x in E] + [np_(u)], _parse_stats(st)

    whole, _ = build(0, T, s0, guess)
    for lo, hi in ((0, T // 3), (T // 3, 2 * T // 3 + 1), (T - 7, T)):
        halo = s0 if lo == 0 else guess[lo - 1]
        part, stats = build(lo, hi - lo, halo, guess[lo:hi])
        for a, b in zip(part, whole):
            np.testing.assert_array_equal(a, b[lo:hi])
        assert stats[0] >= 2 ** 62 and stats[1] >= 2 ** 62  # no bad proposal / step inside the range


def test_streamed_shard_path_matches_run_deer(cuda_device):
    # the sharded driver's streamed-engine path (register systems) at world size 1
    from paper_2508_18413_b200.sharded import run_deer_sharded

    k = cs.GibbsKernel(cs.generate_eight_schools(), seed=0, T=20_000, dtype=torch.float32)
    cfg = cs.DeerConfig(mode="diag-stochastic", hutchinson_samples=3, preconditioner=k.recommended_preconditioner())
    ref = cs.run_deer(k, k.initial_state(), cfg)
    r = run_deer_sharded(k, k.initial_state(), cfg)
    assert r.stats["path"] == "sharded-streamed"
    assert r.iterations == ref.iterations and r.converged == ref.converged
    np.testing.assert_array_equal(np_(r.per_step_converged_at), np_(ref.per_step_converged_at))
    np.testing.assert_allclose(np_(r.trace), np_(ref.trace), rtol=1e-5, atol=1e-5)


@pytest.mark.parametrize("which", ["hmc_diag", "mala_dense12"])
def test_sharded_driver_over_nccl_single_rank(cuda_device, which):
    # the multi-GPU driver's collectives on device tensors through NCCL (world
    # size 1: the pool has one GPU per box; multi-rank exchange is the gloo suite)
    import socket

    import torch.distributed as dist
    from paper_2508_18413_b200.sharded import gather_trace, run_deer_sharded

    if which == "hmc_diag":
        m = cs.model_logp_grad_hvp(cs.rosenbrock(a=0.0, b=0.1, scale1=1.0, scale2=1.0))
        k, s0, cfg = cs.HmcKernel(m, 0.5, 8, seed=0, T=4000), np.zeros(2), cs.DeerConfig(mode="diag-stochastic", clip=1.0)
    else:
        k = cs.MalaKernel(cs.model_logp_grad_hvp(cs.std_normal(12)), 0.3, seed=2, T=1500)
        s0, cfg = np.zeros(12), cs.DeerConfig(mode="dense")
    ref = cs.run_deer(k, s0, cfg)
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device(cuda_device))
    try:
        assert dist.get_backend() == "nccl"
        r = run_deer_sharded(k, s0, cfg)
        full = gather_trace(r, k.T)
    finally:
        dist.destroy_process_group()
    assert r.iterations == ref.iterations and r.converged == ref.converged
    np.testing.assert_allclose(np_(full), np_(ref.trace), atol=1e-10)


@pytest.mark.parametrize("mode,D,T", [("diag", 4, 7001), ("block", 4, 7001), ("dense", 3, 7001), ("dense", 20, 500),
                                       ("dense", 20, 7001), ("dense", 100, 3000), ("dense", 140, 400)])
def test_scan_aggregate_matches_fold(cuda_device, mode, D, T):
    # cs_scan_aggregate = the composed map of the whole sequence (the shard carry);
    # dense D > 8 folds chunk (T = 500) or group (T = 7001) maps as a DGEMM tree
    from paper_2508_18413_b200.sharded import CudaShardOps, apply_agg

    rng = np.random.default_rng(5)
    tt = lambda x: torch.as_tensor(x, device=cuda_device)
    if mode == "diag":
        el = cs.DiagElements(tt(rng.uniform(-0.9, 0.9, (T, D))), tt(rng.normal(size=(T, D))))
        W, key, s0 = D, "diag-stochastic", rng.normal(size=D)
    elif mode == "block":
        el = cs.Block2x2Elements(*(tt(rng.uniform(-0.6, 0.6, (T, D))) for _ in range(4)), tt(rng.normal(size=(T, 2 * D))))
        W, key, s0 = 2 * D, "block2x2-stochastic", rng.normal(size=2 * D)
    else:
        J = rng.normal(size=(T, D, D))
        J *= (0.9 / np.abs(np.linalg.eigvals(J)).max(axis=-1))[:, None, None]
        el = cs.DenseElements(tt(J), tt(rng.normal(size=(T, D))))
        W, key, s0 = D, "dense", rng.normal(size=D)
    agg = CudaShardOps.__new__(CudaShardOps)
    from paper_2508_18413_b200 import _lib

    agg.lib = _lib
    a = agg.aggregate(el)
    last = cs.parallel_affine_solve(el, tt(s0))[-1]
    np.testing.assert_allclose(np_(apply_agg(key, a, tt(s0))), np_(last), rtol=1e-10, atol=1e-10)


# ---------------------------------------------------------------------------
# full-size row scans: the chained-chunk kernel only walks several rounds, group
# boundaries and partial last chunks at large T (a 444-CTA grid and 224-row stages)


@pytest.mark.parametrize("mode,D,T,dtype", [
    ("diag", 18, 2_000_003, torch.float32),
    ("diag", 1, 8_000_017, torch.float64),
    ("diag", 2, 4_000_037, torch.float32),
    ("diag", 64, 500_009, torch.float32),
    ("block", 7, 1_000_003, torch.float64),
])
def test_row_scan_multi_round_vs_oracle(cuda_device, mode, D, T, dtype):
    rng = np.random.default_rng(T)
    tt = lambda x: torch.as_tensor(x, dtype=dtype, device=cuda_device)
    if mode == "diag":
        j = rng.uniform(-0.95, 0.95, (T, D))
        u = rng.normal(size=(T, D))
        s0 = rng.normal(size=D)
        want = O.parallel_affine_solve(O.DiagElements(j, u), s0, workers=16)
        got = np_(cs.parallel_affine_solve(cs.DiagElements(tt(j), tt(u)), tt(s0)))
    else:
        a, b, c, d = (rng.uniform(-0.65, 0.65, (T, D)) for _ in range(4))
        u = rng.normal(size=(T, 2 * D))
        s0 = rng.normal(size=2 * D)
        want = O.parallel_affine_solve(O.Block2x2Elements(a, b, c, d, u), s0, workers=16)
        got = np_(cs.parallel_affine_solve(cs.Block2x2Elements(tt(a), tt(b), tt(c), tt(d), tt(u)), tt(s0)))
    tol = 1e-11 if dtype == torch.float64 else 2e-5
    np.testing.assert_allclose(got, want, atol=tol * 10, rtol=tol)


@pytest.mark.parametrize("case", ["unit", "near_unit", "growing", "zero_entry"])
@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_diag_scan_local_fixup_extremes(cuda_device, case, dtype):
    # the default plain diag scan scans each CTA range from zero and adds
    # P_t e_g while P = prod a is nonzero: maps that never contract (j = 1, j
    # near 1, |j| > 1 in stretches) fix up whole ranges; e = 0 must not turn an
    # overflowing P into NaN.  Against the sequential recursion in f64.
    T, D = 2_200_011, 3  # above the local scan's 2^21 threshold
    rng = np.random.default_rng(11)
    if case == "unit":
        j = np.ones((T, D))
    elif case == "near_unit":
        j = rng.uniform(0.9995, 1.0, (T, D))
    elif case == "growing":
        j = np.where(rng.uniform(size=(T, D)) < 0.5, 1.0005, 0.9995)
    else:
        j = rng.uniform(-0.9, 0.9, (T, D))
    u = rng.normal(size=(T, D)) * (1e-3 if case != "zero_entry" else 1.0)
    s0 = np.zeros(D) if case == "zero_entry" else rng.normal(size=D)
    tt = lambda x: torch.as_tensor(x, dtype=dtype, device=cuda_device)
    jd, ud, sd = (np_(tt(x)).astype(np.float64) for x in (j, u, s0))
    want = O.parallel_affine_solve(O.DiagElements(jd, ud), sd, workers=8)
    got = np_(cs.parallel_affine_solve(cs.DiagElements(tt(j), tt(u)), tt(s0)))
    assert np.all(np.isfinite(got))
    tol = 1e-9 if dtype == torch.float64 else 2e-4
    np.testing.assert_allclose(got, want, rtol=tol, atol=tol * max(1.0, float(np.abs(want).max())))
    again = cs.parallel_affine_solve(cs.DiagElements(tt(j), tt(u)), tt(s0))
    assert torch.equal(again, tt(got)) or np.array_equal(np_(again), got)


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_block_scan_local_fixup_rotation(cuda_device, dtype):
    # block2x2 local scan + fix-up with maps that never contract (rotations,
    # |det| = 1, like a leapfrog step): every range is fixed up end to end
    T, D = 1_100_003, 2
    rng = np.random.default_rng(5)
    th = rng.uniform(-0.05, 0.05, (T, D))
    a, b, c, d = np.cos(th), -np.sin(th), np.sin(th), np.cos(th)
    u = rng.normal(size=(T, 2 * D)) * 1e-3
    s0 = rng.normal(size=2 * D)
    tt = lambda x: torch.as_tensor(x, dtype=dtype, device=cuda_device)
    ad, bd, cd, dd, ud, sd = (np_(tt(x)).astype(np.float64) for x in (a, b, c, d, u, s0))
    want = O.parallel_affine_solve(O.Block2x2Elements(ad, bd, cd, dd, ud), sd, workers=8)
    got = np_(cs.parallel_affine_solve(cs.Block2x2Elements(tt(a), tt(b), tt(c), tt(d), tt(u)), tt(s0)))
    tol = 1e-9 if dtype == torch.float64 else 5e-4
    np.testing.assert_allclose(got, want, rtol=tol, atol=tol * max(1.0, float(np.abs(want).max())))


@pytest.mark.gpu
@pytest.mark.parametrize("D,T", [(1, 3_000_017), (2, 1_000_003), (4, 700_001), (2, 3071), (4, 5)])
def test_small_d_row_scan_coalesced_path(cuda_device, D, T):
    """Small-D fp32 diag scans load stages with 16-byte loads transposed through
    shared memory when j and u are 16-byte aligned; a one-row storage offset takes
    the per-column path.  Same per-segment arithmetic order: bit-identical."""
    rng = np.random.default_rng(D * 1000 + T)
    j = rng.uniform(-0.95, 0.95, (T + 1, D))
    u = rng.normal(size=(T + 1, D))
    s0 = rng.normal(size=D)
    jt = torch.as_tensor(j, dtype=torch.float32, device=cuda_device)
    ut = torch.as_tensor(u, dtype=torch.float32, device=cuda_device)
    s0t = torch.as_tensor(s0, dtype=torch.float32, device=cuda_device)
    aligned = cs.parallel_affine_solve(cs.DiagElements(jt[:T].clone(), ut[:T].clone()), s0t)
    # one-float storage offset (misaligned for 16-byte loads at every D)
    js, us = jt.reshape(-1)[1:1 + T * D].view(T, D), ut.reshape(-1)[1:1 + T * D].view(T, D)
    assert js.data_ptr() % 16 != 0 and us.data_ptr() % 16 != 0
    shifted = cs.parallel_affine_solve(cs.DiagElements(js, us), s0t)
    ref_shift = cs.parallel_affine_solve(cs.DiagElements(js.clone(), us.clone()), s0t)
    assert torch.equal(shifted, ref_shift)
    want = O.parallel_affine_solve(O.DiagElements(j[:T].astype(np.float32).astype(np.float64),
                                                  u[:T].astype(np.float32).astype(np.float64)), s0.astype(np.float32), workers=16)
    np.testing.assert_allclose(np_(aligned), want, atol=2e-4, rtol=2e-5)


@pytest.mark.parametrize("D,misalign,T", [(18, False, 3_000_001), (1, False, 3_000_001), (2, False, 3_000_001),
                                         (4, False, 3_000_001), (2, True, 3_000_001), (4, True, 3_000_001),
                                         (18, False, 4_200_001), (2, True, 4_200_001)])
def test_update_scan_bookkeeping_multi_round(cuda_device, D, misalign, T):
    # the replay's fused bookkeeping (deer.py:273-277) at a multi-round size:
    # last_fail stamps, fail_rows and dmax against a direct evaluation.  D = 1,
    # 2, 4 take the coalesced 16-byte stage loads; a one-float offset of j and
    # u forces the per-column fallback, ragged last stage included.  By default
    # these run the reduce-then-replay kernels (the variant run below covers the
    # two-pass and local-scan kernels)
    from paper_2508_18413_b200 import _lib

    lib = _lib.load()
    it = 7
    g = torch.Generator(device=cuda_device).manual_seed(3 + D)
    off = 1 if misalign else 0
    jb = (torch.rand((T * D + off,), generator=g, device=cuda_device) * 1.9 - 0.95).float()
    ub = torch.randn((T * D + off,), generator=g, device=cuda_device).float()
    j, u = jb[off:].view(T, D), ub[off:].view(T, D)
    s0 = torch.zeros(D, device=cuda_device)
    ref = cs.parallel_affine_solve(cs.DiagElements(j, u), s0)
    guess = ref + torch.randn((T, D), generator=g, device=cuda_device) * 1e-4 * (torch.rand((T, 1), generator=g, device=cuda_device) < 0.3)
    out = torch.empty_like(ref)
    last_fail = torch.full((T,), 2, dtype=torch.int32, device=cuda_device)
    stats = torch.zeros(40, dtype=torch.uint8, device=cuda_device)
    wsb = lib.cs_scan_workspace_bytes(_lib.CS_MODE_DIAG, _lib.CS_F32, T, D)
    ws = torch.empty(wsb, dtype=torch.uint8, device=cuda_device)
    atol, rtol = 1e-5, 1e-5
    _lib.check(lib.cs_scan_diag_update(_lib.CS_F32, _lib.ptr(j), _lib.ptr(u), _lib.ptr(s0), _lib.ptr(out), T, D,
                                       _lib.ptr(ws), wsb, _lib.ptr(guess), atol, rtol, it, _lib.ptr(last_fail),
                                       _lib.ptr(stats), _lib.stream_ptr()))
    torch.cuda.synchronize()
    torch.testing.assert_close(out, ref, atol=1e-5, rtol=1e-5)
    gap = (out.double() - guess.double()).abs()
    fail = (gap > atol + rtol * out.double().abs()).any(dim=1)
    want_lf = torch.where(fail, torch.tensor(it, dtype=torch.int32, device=cuda_device), torch.tensor(2, dtype=torch.int32, device=cuda_device))
    assert torch.equal(last_fail, want_lf)
    raw = stats.cpu().numpy().tobytes()
    fail_rows = int(np.frombuffer(raw[28:32], dtype=np.uint32)[0])
    dmax = float(np.frombuffer(raw[32:40], dtype=np.float64)[0])
    assert fail_rows == int(fail.sum())
    assert dmax == float(gap.max())


@pytest.mark.parametrize("D,T,dtype", [(100, 100_000, torch.float64), (100, 70_001, torch.float32),
                                       (256, 65_537, torch.float64), (65, 131_075, torch.float32)])
def test_wide_reduce_replay_scans(cuda_device, D, T, dtype):
    # 64 < D <= 256: reduce-then-replay for plain and update scans (one to four
    # threads per column; cfg 3 diag's update scan is D = 100, f64) against the
    # oracle scan and a direct evaluation of the bookkeeping
    from paper_2508_18413_b200 import _lib

    lib = _lib.load()
    rng = np.random.default_rng(D + T)
    j = rng.uniform(-0.999, 0.999, (T, D))
    u = rng.normal(size=(T, D))
    s0 = rng.normal(size=D)
    cast = (lambda x: x.astype(np.float32).astype(np.float64)) if dtype == torch.float32 else (lambda x: x)
    want = O.parallel_affine_solve(O.DiagElements(cast(j), cast(u)), cast(s0), workers=16)
    tt = lambda x: torch.as_tensor(x, dtype=dtype, device=cuda_device)
    jt, ut, s0t = tt(j), tt(u), tt(s0)
    tol = dict(atol=1e-9, rtol=1e-9) if dtype == torch.float64 else dict(atol=3e-4, rtol=1e-4)
    plain = cs.parallel_affine_solve(cs.DiagElements(jt, ut), s0t)
    np.testing.assert_allclose(np_(plain), want, **tol)
    g = torch.Generator(device=cuda_device).manual_seed(D)
    wt = torch.as_tensor(want, device=cuda_device)
    guess = (wt + torch.randn((T, D), generator=g, device=cuda_device, dtype=torch.float64) * 1e-4 *
             (torch.rand((T, 1), generator=g, device=cuda_device) < 0.3)).to(dtype)
    out = torch.empty_like(jt)
    lf = torch.full((T,), 1, dtype=torch.int32, device=cuda_device)
    st = torch.zeros(40, dtype=torch.uint8, device=cuda_device)
    code = _lib.CS_F64 if dtype == torch.float64 else _lib.CS_F32
    wsb = lib.cs_scan_workspace_bytes(_lib.CS_MODE_DIAG, code, T, D)
    ws = torch.empty(wsb, dtype=torch.uint8, device=cuda_device)
    atol, rtol = 1e-5, 1e-5
    _lib.check(lib.cs_scan_diag_update(code, _lib.ptr(jt), _lib.ptr(ut), _lib.ptr(s0t), _lib.ptr(out), T, D,
                                       _lib.ptr(ws), wsb, _lib.ptr(guess), atol, rtol, 6, _lib.ptr(lf),
                                       _lib.ptr(st), _lib.stream_ptr()))
    torch.cuda.synchronize()
    np.testing.assert_allclose(np_(out), want, **tol)
    gap = (out.double() - guess.double()).abs()
    fail = (gap > atol + rtol * out.double().abs()).any(dim=1)
    want_lf = torch.where(fail, torch.tensor(6, dtype=torch.int32, device=cuda_device),
                          torch.tensor(1, dtype=torch.int32, device=cuda_device))
    assert torch.equal(lf, want_lf)
    raw = st.cpu().numpy().tobytes()
    assert int(np.frombuffer(raw[28:32], dtype=np.uint32)[0]) == int(fail.sum())
    assert float(np.frombuffer(raw[32:40], dtype=np.float64)[0]) == float(gap.max())


def test_update_scan_rejects_out_overlapping_guess(cuda_device):
    # the update kernels read guess through the read-only path while writing out
    from paper_2508_18413_b200 import _lib

    lib = _lib.load()
    T, D = 1000, 4
    j = torch.full((T, D), 0.5, device=cuda_device)
    u = torch.ones((T, D), device=cuda_device)
    s0 = torch.zeros(D, device=cuda_device)
    g = torch.zeros((T, D), device=cuda_device)
    lf = torch.zeros(T, dtype=torch.int32, device=cuda_device)
    st = torch.zeros(40, dtype=torch.uint8, device=cuda_device)
    wsb = lib.cs_scan_workspace_bytes(_lib.CS_MODE_DIAG, _lib.CS_F32, T, D)
    ws = torch.empty(wsb, dtype=torch.uint8, device=cuda_device)
    rc = lib.cs_scan_diag_update(_lib.CS_F32, _lib.ptr(j), _lib.ptr(u), _lib.ptr(s0), _lib.ptr(g), T, D, _lib.ptr(ws),
                                 wsb, _lib.ptr(g), 1e-5, 1e-5, 1, _lib.ptr(lf), _lib.ptr(st), _lib.stream_ptr())
    assert rc == _lib.CS_ERR_CONFIG


@pytest.mark.parametrize("kind,T", [("slow", 1_000_003), ("slow", 70_001), ("unit", 300_001), ("growing", 250_001),
                                    ("zero_entry", 500_001), ("mixed", 2_000_003), ("mixed", 65_537)])
def test_update_scan_reduce_replay_extremes(cuda_device, kind, T):
    # the reduce-then-replay update scan (2^16 <= T < 2^22): maps that contract
    # slowly (the Newton iterates of cfg 5), not at all, grow for a stretch or
    # hold an exact zero -- states against the f64 oracle scan, bookkeeping
    # against a direct evaluation
    from paper_2508_18413_b200 import _lib

    lib = _lib.load()
    D, it = 18, 4
    rng = np.random.default_rng(T % 1000 + len(kind))
    if kind == "slow":
        j = rng.uniform(0.9990, 0.99999, (T, D))
    elif kind == "unit":
        j = np.ones((T, D))
    elif kind == "growing":
        j = rng.uniform(0.5, 0.95, (T, D))
        j[T // 3:T // 3 + 300] = 1.02
    elif kind == "zero_entry":
        j = rng.uniform(-0.99, 0.99, (T, D))
        j[T // 2, 3] = 0.0
    else:
        j = np.where(rng.uniform(size=(T, D)) < 0.5, rng.uniform(0.999, 1.0, (T, D)), rng.uniform(-0.9, 0.9, (T, D)))
    u = rng.normal(size=(T, D)) * (1e-3 if kind in ("unit", "slow") else 1.0)
    j32, u32 = j.astype(np.float32), u.astype(np.float32)
    s0 = rng.normal(size=D).astype(np.float32)
    want = O.parallel_affine_solve(O.DiagElements(j32.astype(np.float64), u32.astype(np.float64)),
                                   s0.astype(np.float64), workers=16)
    jt, ut = torch.as_tensor(j32, device=cuda_device), torch.as_tensor(u32, device=cuda_device)
    s0t = torch.as_tensor(s0, device=cuda_device)
    wt = torch.as_tensor(want, device=cuda_device)
    g = torch.Generator(device=cuda_device).manual_seed(T)
    guess = (wt + torch.randn((T, D), generator=g, device=cuda_device, dtype=torch.float64) * 1e-4 *
             (torch.rand((T, 1), generator=g, device=cuda_device) < 0.3)).float()
    out = torch.empty_like(jt)
    last_fail = torch.full((T,), 1, dtype=torch.int32, device=cuda_device)
    stats = torch.zeros(40, dtype=torch.uint8, device=cuda_device)
    wsb = lib.cs_scan_workspace_bytes(_lib.CS_MODE_DIAG, _lib.CS_F32, T, D)
    ws = torch.empty(wsb, dtype=torch.uint8, device=cuda_device)
    atol, rtol = 1e-5, 1e-5
    _lib.check(lib.cs_scan_diag_update(_lib.CS_F32, _lib.ptr(jt), _lib.ptr(ut), _lib.ptr(s0t), _lib.ptr(out), T, D,
                                       _lib.ptr(ws), wsb, _lib.ptr(guess), atol, rtol, it, _lib.ptr(last_fail),
                                       _lib.ptr(stats), _lib.stream_ptr()))
    torch.cuda.synchronize()
    scale = np.abs(want).max()
    np.testing.assert_allclose(np_(out), want, atol=2e-5 * max(scale, 1.0) * (30 if kind == "unit" else 1), rtol=1e-4)
    gap = (out.double() - guess.double()).abs()
    fail = (gap > atol + rtol * out.double().abs()).any(dim=1)
    want_lf = torch.where(fail, torch.tensor(it, dtype=torch.int32, device=cuda_device),
                          torch.tensor(1, dtype=torch.int32, device=cuda_device))
    assert torch.equal(last_fail, want_lf)
    raw = stats.cpu().numpy().tobytes()
    assert int(np.frombuffer(raw[28:32], dtype=np.uint32)[0]) == int(fail.sum())
    assert float(np.frombuffer(raw[32:40], dtype=np.float64)[0]) == float(gap.max())
    # the plain scan of the same maps (below 2^20 the reduce-then-replay kernels, above the local scan)
    plain = cs.parallel_affine_solve(cs.DiagElements(jt, ut), s0t)
    np.testing.assert_allclose(np_(plain), want, atol=2e-5 * max(scale, 1.0) * (30 if kind == "unit" else 1), rtol=1e-4)
    # run to run: bit-identical
    out2 = torch.empty_like(out)
    _lib.check(lib.cs_scan_diag_update(_lib.CS_F32, _lib.ptr(jt), _lib.ptr(ut), _lib.ptr(s0t), _lib.ptr(out2), T, D,
                                       _lib.ptr(ws), wsb, _lib.ptr(guess), atol, rtol, it, _lib.ptr(last_fail),
                                       _lib.ptr(stats), _lib.stream_ptr()))
    torch.cuda.synchronize()
    assert torch.equal(out, out2)


@pytest.mark.skipif(bool(__import__("os").environ.get("CS_SCAN_LBW")), reason="already the variant run")
@pytest.mark.parametrize("lag,round_kb", [(1, 4096), (2, 16384)])
def test_row_scan_lookback_warp_variant(cuda_device, lag, round_kb):
    # the opt-in row-scan variant with dedicated look-back and publisher warps
    # (CS_SCAN_LBW=1; the switch is read once per process, hence a subprocess):
    # the multi-round parity and fused-bookkeeping cases above, many small rounds
    import os
    import subprocess
    import sys

    # (CS_SCAN_RR=0: the update cases take the two-pass kernel below 2^22 and the
    # local scan + fix-up with per-tile bookkeeping above)
    env = dict(os.environ, CS_SCAN_LBW="1", CS_SCAN_LAG=str(lag), CS_SCAN_ROUND_KB=str(round_kb), CS_SCAN_RR="0")
    r = subprocess.run([sys.executable, "-m", "pytest", os.path.abspath(__file__), "-x", "-q", "-m", "gpu", "-p",
                        "no:cacheprovider", "-k", "multi_round or update_scan_bookkeeping or scan_kats or diag_and_block"],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


@pytest.mark.parametrize("T", [1, 2, 17, 100, 127, 128, 129])
@pytest.mark.parametrize("D", [65, 300])
@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_wide_short_scans_vs_oracle(cuda_device, T, D, dtype):
    # scan_cols_small (D > 64, T <= 128: one CTA per column block, no look-back) and
    # scan_cols just above the switch, diag and block2x2
    rng = np.random.default_rng(1000 * T + D)
    tt = lambda x: torch.as_tensor(x, dtype=dtype, device=cuda_device)
    tol = 1e-12 if dtype == torch.float64 else 2e-5
    j, u, s0 = rng.uniform(-0.95, 0.95, (T, D)), rng.normal(size=(T, D)), rng.normal(size=D)
    want = O.parallel_affine_solve(O.DiagElements(j, u), s0, workers=4)
    got = np_(cs.parallel_affine_solve(cs.DiagElements(tt(j), tt(u)), tt(s0)))
    np.testing.assert_allclose(got, want, atol=tol * 10, rtol=tol)
    a, b, c, d = (rng.uniform(-0.65, 0.65, (T, D)) for _ in range(4))
    ub, s0b = rng.normal(size=(T, 2 * D)), rng.normal(size=2 * D)
    want = O.parallel_affine_solve(O.Block2x2Elements(a, b, c, d, ub), s0b, workers=4)
    got = np_(cs.parallel_affine_solve(cs.Block2x2Elements(tt(a), tt(b), tt(c), tt(d), tt(ub)), tt(s0b)))
    np.testing.assert_allclose(got, want, atol=tol * 10, rtol=tol)


def test_wide_short_update_scan_bookkeeping(cuda_device):
    # the small-T kernel's fused bookkeeping against a direct evaluation
    from paper_2508_18413_b200 import _lib

    lib = _lib.load()
    T, D, it = 100, 1000, 5
    g = torch.Generator(device=cuda_device).manual_seed(9)
    a, b, c, d = ((torch.rand((T, D), generator=g, device=cuda_device, dtype=torch.float64) * 1.3 - 0.65)
                  for _ in range(4))
    u = torch.randn((T, 2 * D), generator=g, device=cuda_device, dtype=torch.float64)
    s0 = torch.zeros(2 * D, device=cuda_device, dtype=torch.float64)
    ref = cs.parallel_affine_solve(cs.Block2x2Elements(a, b, c, d, u), s0)
    guess = ref + torch.randn((T, 2 * D), generator=g, device=cuda_device, dtype=torch.float64) * 1e-3 * (
        torch.rand((T, 1), generator=g, device=cuda_device) < 0.4)
    out = torch.empty_like(ref)
    last_fail = torch.full((T,), 3, dtype=torch.int32, device=cuda_device)
    stats = torch.zeros(40, dtype=torch.uint8, device=cuda_device)
    wsb = lib.cs_scan_workspace_bytes(_lib.CS_MODE_BLOCK, _lib.CS_F64, T, D)
    ws = torch.empty(wsb, dtype=torch.uint8, device=cuda_device)
    atol, rtol = 1e-6, 1e-6
    _lib.check(lib.cs_scan_block_update(_lib.CS_F64, *[_lib.ptr(x) for x in (a, b, c, d, u, s0, out)], T, D,
                                        _lib.ptr(ws), wsb, _lib.ptr(guess), atol, rtol, it, _lib.ptr(last_fail),
                                        _lib.ptr(stats), _lib.stream_ptr()))
    torch.cuda.synchronize()
    torch.testing.assert_close(out, ref, atol=1e-12, rtol=1e-12)
    gap = (out - guess).abs()
    fail = (gap > atol + rtol * out.abs()).any(dim=1)
    want_lf = torch.where(fail, torch.tensor(it, dtype=torch.int32, device=cuda_device),
                          torch.tensor(3, dtype=torch.int32, device=cuda_device))
    assert torch.equal(last_fail, want_lf)
    raw = stats.cpu().numpy().tobytes()
    assert (int(np.frombuffer(raw[28:32], dtype=np.uint32)[0]) > 0) == bool(fail.any())
    assert float(np.frombuffer(raw[32:40], dtype=np.float64)[0]) == float(gap.max())


@pytest.mark.parametrize("case", ["hmc-diag", "gibbs-diag3", "leapfrog-block", "mala-mog-diag"])
def test_streamed_window_matches_host_window(cuda_device, case):
    # deer.py:287-319 on the device engine against the host-driven window loop:
    # same iterations, delta history, per-step records and trace
    if case == "hmc-diag":
        m = cs.model_logp_grad_hvp(cs.rosenbrock(a=0.0, b=0.1, scale1=1.0, scale2=1.0))
        k, s0 = cs.HmcKernel(m, 0.5, 8, seed=0, T=3000), np.zeros(2)
        kw = dict(mode="diag-stochastic", clip=1.0, window_len=500, max_iters=2000)
    elif case == "gibbs-diag3":
        k = cs.GibbsKernel(cs.generate_eight_schools(), seed=0, T=4000)
        s0 = k.initial_state()
        kw = dict(mode="diag-stochastic", hutchinson_samples=3, preconditioner=k.recommended_preconditioner(),
                  window_len=1000, max_iters=4000)
    elif case == "leapfrog-block":
        tg = cs.gaussian(np.array([0.5, -0.5]), np.array([[1.2, 0.0], [0.7, 0.6]]))
        k = cs.LeapfrogSystem(cs.model_logp_grad_hvp(tg), 0.1, 300)
        s0 = np.array([0.5, -0.5, 0.2, 0.1])
        kw = dict(mode="block2x2-stochastic", window_len=64, max_iters=500)
    else:
        k = cs.MalaKernel(cs.model_logp_grad_hvp(cs.mog()), 0.1, seed=1, T=4096)
        s0 = np.zeros(2)
        kw = dict(mode="diag-stochastic", clip=1.0, window_len=512, max_iters=4000)
    a = cs.run_deer(k, s0, cs.DeerConfig(**kw))
    b = cs.run_deer(k, s0, cs.DeerConfig(engine="host", **kw))
    assert a.stats["path"] == "streamed-window" and b.stats["path"] == "host"
    assert a.iterations == b.iterations and a.converged == b.converged
    np.testing.assert_array_equal(np_(a.per_step_converged_at), np_(b.per_step_converged_at))
    np.testing.assert_allclose(a.delta_history, b.delta_history, rtol=1e-5, atol=1e-12)
    np.testing.assert_allclose(np_(a.trace), np_(b.trace), rtol=1e-6, atol=1e-8)

"""The reference's target-model tests (test_targets.py:60-255) against this
package's device models; CSV ingestion (test_targets.py:170-227) is out of
scope and the basis/transform tests live in test_basis.py."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

cs = pytest.importorskip("paper_2508_18413_b200")
T_ = cs.targets


def np_(t):
    return t.detach().cpu().numpy() if torch.is_tensor(t) else np.asarray(t)


def fd_grad(logp, x, h=1e-4):  # test_targets.py:28-34
    g = np.empty_like(x)
    for i in range(x.size):
        e = np.zeros_like(x)
        e[i] = h
        g[i] = (float(logp(x + e)) - float(logp(x - e))) / (2 * h)
    return g


def fd_hvp(grad, x, v, h=1e-5):
    return (np_(grad(x + h * v)) - np_(grad(x - h * v))) / (2 * h)


def rel_err(got, want):
    got, want = np_(got), np_(want)
    return np.linalg.norm(got - want) / max(1.0, np.linalg.norm(want))


def make_specs():  # test_targets.py:45-56
    rng = np.random.default_rng(0)
    L = np.tril(0.3 * rng.normal(size=(4, 4))) + np.eye(4)
    Xd = rng.normal(size=(30, 3))
    yd = (rng.uniform(size=30) < 0.5).astype(float)
    return {"std-normal": (T_.std_normal(4), 1.5), "gaussian": (T_.gaussian(rng.normal(size=4), L), 1.5),
            "rosenbrock": (T_.rosenbrock(), 1.0), "mog": (T_.mog(), 3.0),
            "blr": (T_.blr(Xd, yd, prior_precision=0.5), 1.0)}


@pytest.mark.parametrize("name", ["std-normal", "gaussian", "rosenbrock", "mog", "blr"])
def test_grad_and_hvp_match_finite_differences(cuda_device, name):  # test_targets.py:59-70
    spec, scale = make_specs()[name]
    model = T_.model_logp_grad_hvp(spec)
    rng = np.random.default_rng(sum(map(ord, name)))
    for _ in range(25):
        x = scale * rng.normal(size=model.dim)
        assert rel_err(model.grad(x), fd_grad(model.logp, x)) <= 1e-5
        v = rng.normal(size=model.dim)
        v /= np.linalg.norm(v)
        assert rel_err(model.hvp(x, v), fd_hvp(model.grad, x, v)) <= 1e-5


@pytest.mark.parametrize("name", ["gaussian", "rosenbrock", "mog", "blr"])
def test_hvp_linear_in_v(cuda_device, name):  # test_targets.py:73-82
    spec, scale = make_specs()[name]
    model = T_.model_logp_grad_hvp(spec)
    rng = np.random.default_rng(1)
    x = scale * rng.normal(size=model.dim)
    v1, v2 = rng.normal(size=model.dim), rng.normal(size=model.dim)
    lhs = np_(model.hvp(x, 2.0 * v1 - 0.5 * v2))
    rhs = 2.0 * np_(model.hvp(x, v1)) - 0.5 * np_(model.hvp(x, v2))
    np.testing.assert_allclose(lhs, rhs, atol=1e-10)


def test_std_normal_closed_form(cuda_device):  # test_targets.py:85-91
    model = T_.model_logp_grad_hvp(T_.std_normal(3))
    x, v = np.array([1.0, -2.0, 0.5]), np.array([0.3, 0.0, -1.0])
    np.testing.assert_array_equal(np_(model.grad(x)), -x)
    np.testing.assert_array_equal(np_(model.hvp(x, v)), -v)
    assert float(model.logp(x)) == -0.5 * np.dot(x, x)


def test_batched_evaluation_matches_loop(cuda_device):  # test_targets.py:94-108
    model = T_.model_logp_grad_hvp(make_specs()["mog"][0])
    rng = np.random.default_rng(2)
    X, V = rng.normal(size=(7, 5, 2)) * 3, rng.normal(size=(7, 5, 2))
    lp, g, hv = np_(model.logp(X)), np_(model.grad(X)), np_(model.hvp(X, V))
    assert lp.shape == (7, 5) and g.shape == (7, 5, 2)
    for i in range(7):
        for j in range(5):
            assert lp[i, j] == pytest.approx(float(model.logp(X[i, j])), abs=1e-12)
            np.testing.assert_allclose(g[i, j], np_(model.grad(X[i, j])), atol=1e-12)
            np.testing.assert_allclose(hv[i, j], np_(model.hvp(X[i, j], V[i, j])), atol=1e-12)


def test_blr_toy_hvp_against_grad_differences(cuda_device):  # test_targets.py:111-117
    X = np.array([[1.0, 0.0], [0.5, -1.0], [2.0, 1.0]])
    y = np.array([1.0, 0.0, 1.0])
    model = T_.model_logp_grad_hvp(T_.blr(X, y, prior_precision=1.0))
    beta, e1 = np.array([0.3, -0.2]), np.array([1.0, 0.0])
    assert rel_err(model.hvp(beta, e1), fd_hvp(model.grad, beta, e1)) <= 1e-5


def test_mog_logp_finite_far_out(cuda_device):  # test_targets.py:120-127
    model = T_.model_logp_grad_hvp(T_.mog())
    grid = np.stack(np.meshgrid(np.linspace(-13, 13, 41), np.linspace(-13, 13, 41)), axis=-1)
    assert np.all(np.isfinite(np_(model.logp(grid)))) and np.all(np.isfinite(np_(model.grad(grid))))


def test_blr_large_batch_matches_one_shot_formula(cuda_device):  # test_targets.py:130-148
    rng = np.random.default_rng(3)
    X = rng.normal(size=(50, 4))
    y = (rng.uniform(size=50) < 0.5).astype(float)
    model = T_.model_logp_grad_hvp(T_.blr(X, y))
    B = rng.normal(size=(997, 4))
    eta = B @ X.T
    want = eta @ y - np.logaddexp(0.0, eta).sum(-1) - 0.5 * np.sum(B * B, -1)
    np.testing.assert_allclose(np_(model.logp(B)), want, atol=1e-10)
    gwant = (y - 1.0 / (1.0 + np.exp(-eta))) @ X - B
    np.testing.assert_allclose(np_(model.grad(B)), gwant, atol=1e-10)


@pytest.mark.parametrize("D", [3, 100, 300])
def test_gemm_targets_native_match_numpy(cuda_device, D):
    # logistic regression and dense Gaussians evaluate on the library's DMMA GEMM
    # (cs_target_eval): logp / grad / hvp against the numpy formulas
    # (targets.py:160-287), including a broadcast tangent and a leading batch shape
    rng = np.random.default_rng(D)
    X = rng.normal(size=(257, D)) / np.sqrt(D)
    y = (rng.uniform(size=257) < 0.5).astype(float)
    blr = T_.model_logp_grad_hvp(T_.blr(X, y, prior_precision=0.7))
    B = rng.normal(size=(2, 33, D))
    V = rng.normal(size=D)
    eta = B @ X.T
    p = 1.0 / (1.0 + np.exp(-eta))
    np.testing.assert_allclose(np_(blr.logp(B)), eta @ y - np.logaddexp(0.0, eta).sum(-1) - 0.35 * np.sum(B * B, -1),
                               rtol=1e-12, atol=1e-10)
    np.testing.assert_allclose(np_(blr.grad(B)), (y - p) @ X - 0.7 * B, rtol=1e-12, atol=1e-10)
    np.testing.assert_allclose(np_(blr.hvp(B, V)), -(((p * (1 - p)) * (V @ X.T)) @ X) - 0.7 * V,
                               rtol=1e-12, atol=1e-10)
    Q, _ = np.linalg.qr(rng.normal(size=(D, D)))
    Lc = np.linalg.cholesky((Q * np.exp(rng.uniform(-1, 1, D))) @ Q.T)
    mu = rng.normal(size=D)
    g = T_.model_logp_grad_hvp(T_.gaussian(mu, Lc))
    P = Lc @ Lc.T
    h = (B - mu) @ Lc
    np.testing.assert_allclose(np_(g.logp(B)), -0.5 * np.sum(h * h, -1), rtol=1e-12, atol=1e-9)
    np.testing.assert_allclose(np_(g.grad(B)), -((B - mu) @ P), rtol=1e-12, atol=1e-9)
    np.testing.assert_allclose(np_(g.hvp(B, V)), np.broadcast_to(-(V @ P), B.shape), rtol=1e-12, atol=1e-9)
    assert g.logp(B[0, 0]).shape == () and g.grad(B[0, 0]).shape == (D,)


def test_invalid_specs_rejected(cuda_device):  # test_targets.py:151-164
    with pytest.raises(cs.ConfigurationError):
        T_.mog(weights=[0.5, 0.6], means=[[0.0], [1.0]])
    with pytest.raises(cs.ConfigurationError):
        T_.mog(variances=[1.0, 1.0, 1.0, -1.0])
    with pytest.raises(cs.ConfigurationError):
        T_.rosenbrock(scale2=0.0)
    with pytest.raises(cs.ConfigurationError):
        T_.blr(np.zeros((3, 2)), np.array([0.0, 2.0, 1.0]))
    with pytest.raises(cs.ConfigurationError):
        T_.blr(np.zeros((3, 2)), np.zeros(4))
    with pytest.raises(cs.ConfigurationError):
        T_.gaussian(np.zeros(2), -np.eye(2))


def test_synthetic_dataset_deterministic(cuda_device):  # test_targets.py:230-237
    Xa, ya, ba = T_.synthetic_credit_like()
    Xb, yb, bb = T_.synthetic_credit_like()
    assert Xa.shape == (1000, 25) and ya.shape == (1000,)
    np.testing.assert_array_equal(Xa, Xb)
    np.testing.assert_array_equal(ya, yb)
    np.testing.assert_array_equal(ba, bb)
    assert set(np.unique(ya)) <= {0.0, 1.0}


def test_map_estimate_recovers_signs(cuda_device):  # test_targets.py:240-252
    from scipy.optimize import minimize

    X, y, beta_star = T_.synthetic_credit_like()
    model = T_.model_logp_grad_hvp(T_.blr(X, y, prior_precision=1.0))
    res = minimize(lambda b: -float(model.logp(b)), np.zeros(25), jac=lambda b: -np_(model.grad(b)),
                   method="L-BFGS-B")
    assert res.success
    assert np.mean(np.sign(res.x) == np.sign(beta_star)) >= 0.9

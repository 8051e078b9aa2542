"""Orthogonal change of basis (targets.py:400-517): the reference's own
test_targets.py basis / transform cases against this package, and a golden
eigenbasis solve made by running the reference (tests/golden/basis.npz)."""

import numpy as np
import pytest
import torch

import paper_2508_18413_b200 as cs
from conftest import golden
from paper_2508_18413_b200.errors import StructuralError

pytestmark = pytest.mark.gpu


def np_(x):
    return x.detach().cpu().numpy() if torch.is_tensor(x) else np.asarray(x)


class NonlinToy(cs.TransitionSystem):
    """s' = tanh(W s) + shift (test_targets.py:296-309)."""

    def __init__(self, W, shift, T=16):
        super().__init__(W.shape[0], cs.NoiseTable(0, {}, T))
        self.W = torch.as_tensor(W, device=self.device)
        self.shift = torch.as_tensor(shift, device=self.device)

    def _step_batch(self, ts, S):
        return torch.tanh(S @ self.W.T) + self.shift

    def _jvp_batch(self, ts, S, V):
        return (1.0 - torch.tanh(S @ self.W.T) ** 2) * (V @ self.W.T)


def make_toy(seed=6, dim=3):
    rng = np.random.default_rng(seed)
    return NonlinToy(0.7 * rng.normal(size=(dim, dim)), rng.normal(size=dim))


def test_jacobi_identity(cuda_device):
    b = cs.orthogonal_basis(np.eye(3))
    np.testing.assert_allclose(np_(b.Q.T @ b.Q), np.eye(3), atol=1e-12)
    np.testing.assert_array_equal(np_(b.eigenvalues), np.ones(3))


def test_jacobi_2x2_closed_form(cuda_device):
    C = np.array([[2.0, 1.0], [1.0, 2.0]])
    b = cs.orthogonal_basis(C)
    np.testing.assert_allclose(np_(b.eigenvalues), [3.0, 1.0], atol=1e-12)
    r = 1.0 / np.sqrt(2.0)
    np.testing.assert_allclose(np.abs(np_(b.Q)), [[r, r], [r, r]], atol=1e-12)
    np.testing.assert_allclose(C @ np_(b.Q), np_(b.Q) * np_(b.eigenvalues), atol=1e-12)


def test_jacobi_reconstruction_random(cuda_device):
    M = np.random.default_rng(5).normal(size=(16, 16))
    C = M + M.T
    b = cs.orthogonal_basis(C)
    Q, e = np_(b.Q), np_(b.eigenvalues)
    assert np.max(np.abs(Q @ np.diag(e) @ Q.T - C)) < 1e-9
    assert np.all(np.diff(e) <= 1e-12)
    assert np.max(np.abs(Q.T @ Q - np.eye(16))) <= 1e-10


def test_basis_matches_the_reference_jacobi(cuda_device):
    g = golden("basis")
    b = cs.orthogonal_basis(g["C"])
    np.testing.assert_allclose(np_(b.eigenvalues), g["eig"], atol=1e-10)
    np.testing.assert_allclose(np_(b.Q), g["Q"], atol=1e-8)  # same ordering and sign convention


def test_jacobi_rejects_asymmetric(cuda_device):
    with pytest.raises(StructuralError):
        cs.orthogonal_basis(np.array([[1.0, 2.0], [0.0, 1.0]]))
    with pytest.raises(StructuralError):
        cs.orthogonal_basis(np.zeros((2, 3)))


def test_identity_transform_is_noop(cuda_device):
    sys_ = make_toy()
    s0 = np.array([0.2, -0.4, 1.0])
    np.testing.assert_allclose(np_(cs.sequential_evaluate(cs.transform_system(sys_, np.eye(3)), s0)),
                               np_(cs.sequential_evaluate(sys_, s0)), atol=1e-14)


def test_permutation_transform_relabels_trace(cuda_device):
    sys_ = make_toy()
    Q = np.eye(3)[:, [2, 0, 1]]
    s0 = np.array([0.2, -0.4, 1.0])
    z = np_(cs.sequential_evaluate(cs.transform_system(sys_, Q), s0 @ Q))
    np.testing.assert_allclose(z, np_(cs.sequential_evaluate(sys_, s0)) @ Q, atol=1e-13)


def test_transform_round_trip_reproduces_trace(cuda_device):
    sys_ = make_toy(seed=8)
    rng = np.random.default_rng(9)
    Q = np.linalg.qr(rng.normal(size=(3, 3)))[0]
    w = cs.transform_system(sys_, Q)
    s0 = rng.normal(size=3)
    z = cs.sequential_evaluate(w, w.transform_state(s0))
    np.testing.assert_allclose(np_(w.untransform_state(z)), np_(cs.sequential_evaluate(sys_, s0)), atol=1e-12)


def test_transformed_jvp_matches_finite_differences(cuda_device):
    sys_ = make_toy(seed=10)
    w = cs.transform_system(sys_, np.linalg.qr(np.random.default_rng(11).normal(size=(3, 3)))[0])
    rng = np.random.default_rng(12)
    z, v = rng.normal(size=3), rng.normal(size=3)
    h = 1e-6
    fd = (np_(w.step(2, z + h * v)) - np_(w.step(2, z - h * v))) / (2 * h)
    np.testing.assert_allclose(np_(w.jvp(2, z, v)), fd, atol=1e-8)


def test_transform_validates_inputs(cuda_device):
    sys_ = make_toy()
    with pytest.raises(StructuralError):
        cs.transform_system(sys_, np.eye(4))
    with pytest.raises(StructuralError):
        cs.transform_system(sys_, np.full((3, 3), 0.5))


def test_eigenbasis_solve_matches_the_reference(cuda_device):
    # diag quasi-Newton MALA on a correlated Gaussian, solved in the precision's
    # eigenbasis: the reference run converges in 11 iterations (51 without it)
    g = golden("basis")
    m = cs.model_logp_grad_hvp(cs.gaussian(np.array([0.5, -1.0, 0.0, 1.0]), g["chol"]))
    k = cs.MalaKernel(m, 0.15, seed=9, T=400)
    w = cs.transform_system(k, cs.orthogonal_basis(g["P"]).Q)
    r = cs.run_deer(w, w.transform_state(np.zeros(4)), cs.DeerConfig(mode="diag-stochastic"))
    assert r.stats["path"] == "streamed"  # Q fused into the element builder, no eager conjugation
    assert r.converged == bool(g["z_converged"]) and r.iterations == int(g["z_iterations"])
    np.testing.assert_allclose(np_(r.trace), g["z_trace"], atol=1e-8, rtol=1e-8)
    np.testing.assert_allclose(np_(w.untransform_state(r.trace)), g["seq"], atol=1e-3, rtol=1e-3)


@pytest.mark.parametrize("kind", ["mala", "hmc"])
def test_fused_basis_matches_eager_conjugation(cuda_device, kind):
    # Q fused into the MALA / HMC kernels against the same conjugation done as
    # batched matmuls around the plain system (targets.py:487-501)
    from paper_2508_18413_b200.basis import _FusedTransformed, _TransformedSystem

    g = golden("basis")
    m = cs.model_logp_grad_hvp(cs.gaussian(np.array([0.5, -1.0, 0.0, 1.0]), g["chol"]))
    k = cs.MalaKernel(m, 0.15, seed=9, T=400) if kind == "mala" else cs.HmcKernel(m, 0.2, 5, seed=9, T=400)
    Q = cs.orthogonal_basis(g["P"]).Q
    fused, eager = cs.transform_system(k, Q), _TransformedSystem(k, Q)
    assert isinstance(fused, _FusedTransformed) and not isinstance(eager, _FusedTransformed)
    rng = np.random.default_rng(4)
    Z = torch.as_tensor(rng.normal(size=(64, 4)), device=cuda_device)
    V = torch.as_tensor(rng.normal(size=(64, 4)), device=cuda_device)
    ts = torch.arange(1, 65, device=cuda_device)
    torch.testing.assert_close(fused.step_batch(ts, Z), eager.step_batch(ts, Z), atol=1e-12, rtol=1e-12)
    torch.testing.assert_close(fused.jvp_batch(ts, Z, V), eager.jvp_batch(ts, Z, V), atol=1e-12, rtol=1e-12)
    z0 = fused.transform_state(np.zeros(4))
    torch.testing.assert_close(cs.sequential_evaluate(fused, z0), cs.sequential_evaluate(eager, z0), atol=1e-10,
                               rtol=1e-10)
    for mode in ("diag-stochastic", "dense"):
        a = cs.run_deer(fused, z0, cs.DeerConfig(mode=mode))
        b = cs.run_deer(eager, z0, cs.DeerConfig(mode=mode))
        assert a.stats["path"] == "streamed" and b.stats["path"] == "host"
        assert a.iterations == b.iterations and a.converged == b.converged
        torch.testing.assert_close(a.trace, b.trace, atol=1e-9, rtol=1e-9)

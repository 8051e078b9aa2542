"""The affine-element API (pscan.py) mirrored case by case from the reference's
own tests/test_pscan.py: monoid laws and structural errors on CPU tensors, and
the CUDA scans against the loop at the reference's sequence lengths."""

import numpy as np
import pytest
import torch

import paper_2508_18413_b200 as cs
from paper_2508_18413_b200.errors import StructuralError

VARIANTS = ["diag", "dense", "block"]


def rand_elements(rng, variant, T, D, device="cpu", dtype=torch.float64):
    tt = lambda x: torch.as_tensor(x, dtype=dtype, device=device)
    if variant == "diag":
        return cs.DiagElements(tt(rng.uniform(-0.9, 0.9, (T, D))), tt(rng.normal(size=(T, D))))
    if variant == "dense":
        return cs.DenseElements(tt(rng.normal(size=(T, D, D)) * (0.9 / (2 * np.sqrt(D)))), tt(rng.normal(size=(T, D))))
    a, b, c, d = (tt(rng.uniform(-0.6, 0.6, (T, D))) for _ in range(4))
    return cs.Block2x2Elements(a, b, c, d, tt(rng.normal(size=(T, 2 * D))))


def block_to_dense(e):
    """Expand block2x2 elements into full (2D x 2D) Jacobians."""
    T, D = e.a.shape
    J = torch.zeros((T, 2 * D, 2 * D), dtype=e.a.dtype)
    idx = torch.arange(D)
    J[:, idx, idx], J[:, idx, D + idx] = e.a, e.b
    J[:, D + idx, idx], J[:, D + idx, D + idx] = e.c, e.d
    return cs.DenseElements(J, e.u.clone())


def as_np(e):
    return [np.asarray(x) for x in (e.j, e.u)] if isinstance(e, cs.DiagElements) else \
        [np.asarray(x) for x in (e.J, e.u)] if isinstance(e, cs.DenseElements) else \
        [np.asarray(x) for x in (e.a, e.b, e.c, e.d, e.u)]


def test_diag_frozen_scalars():  # test_pscan.py:55-62
    e = cs.DiagElements(torch.tensor([[2.0], [3.0], [4.0]]), torch.ones((3, 1)))
    np.testing.assert_array_equal(cs.sequential_affine_solve(e, torch.ones(1)).numpy().ravel(), [3, 10, 41])


def test_dense_compose_frozen():  # test_pscan.py:65-72
    swap = cs.DenseElements(torch.tensor([[0.0, 1.0], [1.0, 0.0]]), torch.tensor([1.0, 0.0]))
    two = cs.DenseElements(2 * torch.eye(2), torch.zeros(2))
    c = cs.compose(two, swap)
    np.testing.assert_array_equal(c.J.numpy(), [[0, 2], [2, 0]])
    np.testing.assert_array_equal(c.u.numpy(), [2, 0])


@pytest.mark.parametrize("variant", VARIANTS)
def test_compose_agrees_with_application(variant):  # test_pscan.py:76-84
    rng = np.random.default_rng(1)
    e1, e2 = rand_elements(rng, variant, 16, 3), rand_elements(rng, variant, 16, 3)
    s = torch.as_tensor(rng.normal(size=(16, e1.dim)))
    torch.testing.assert_close(cs.apply_element(cs.compose(e2, e1), s),
                               cs.apply_element(e2, cs.apply_element(e1, s)), atol=1e-12, rtol=1e-12)


@pytest.mark.parametrize("variant", VARIANTS)
def test_identity_element_is_neutral(variant):  # test_pscan.py:87-95
    rng = np.random.default_rng(2)
    e = rand_elements(rng, variant, 9, 4)
    idn = cs.identity_element(e)
    for got in (cs.compose(idn, e), cs.compose(e, idn)):
        for x, y in zip(as_np(got), as_np(e)):
            np.testing.assert_allclose(x, y, atol=1e-15)


@pytest.mark.parametrize("variant", VARIANTS)
def test_compose_associative(variant):  # test_pscan.py:98-115
    rng = np.random.default_rng(3)
    a, b, c = (rand_elements(rng, variant, 11, 3) for _ in range(3))
    for x, y in zip(as_np(cs.compose(c, cs.compose(b, a))), as_np(cs.compose(cs.compose(c, b), a))):
        np.testing.assert_allclose(x, y, atol=1e-12)


def test_block_compose_matches_dense_expansion():  # test_pscan.py:118-125
    rng = np.random.default_rng(4)
    e1, e2 = rand_elements(rng, "block", 50, 4), rand_elements(rng, "block", 50, 4)
    blk = block_to_dense(cs.compose(e2, e1))
    dense = cs.compose(block_to_dense(e2), block_to_dense(e1))
    np.testing.assert_allclose(blk.J.numpy(), dense.J.numpy(), atol=1e-12)
    np.testing.assert_allclose(blk.u.numpy(), dense.u.numpy(), atol=1e-12)


def test_compose_rejects_mismatches():  # test_pscan.py:128-134
    d = cs.DiagElements(torch.ones(3), torch.zeros(3))
    with pytest.raises(StructuralError):
        cs.compose(d, cs.DenseElements(torch.eye(3), torch.zeros(3)))
    with pytest.raises(StructuralError):
        cs.compose(d, cs.DiagElements(torch.ones(4), torch.zeros(4)))


def test_batch_shape_rejected_by_solver():  # test_pscan.py:244-247
    e = cs.DiagElements(torch.ones((2, 4, 3)), torch.zeros((2, 4, 3)))
    with pytest.raises(StructuralError):
        cs.sequential_affine_solve(e, torch.zeros(3))


def test_default_chunk_layout():  # test_pscan.py:200-203
    assert cs.default_chunk(100, 4) == 100
    assert cs.default_chunk(10_000, 4) == 313
    assert cs.default_chunk(1_000_000, 8) == 15625


# ---------------------------------------------------------------------------
# the CUDA scans


@pytest.mark.gpu
@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("T", [1, 2, 255, 256, 257, 1024])
def test_parallel_matches_sequential(cuda_device, variant, T):  # test_pscan.py:140-148
    rng = np.random.default_rng(100 + T)
    e = rand_elements(rng, variant, T, 4, device=cuda_device)
    s0 = torch.as_tensor(rng.normal(size=e.dim), device=cuda_device)
    want = cs.sequential_affine_solve(e, s0)
    got = cs.parallel_affine_solve(e, s0, workers=4)
    torch.testing.assert_close(got, want, atol=1e-10, rtol=0)


@pytest.mark.gpu
def test_block_solver_matches_dense_expansion_solver(cuda_device):  # test_pscan.py:151-157
    rng = np.random.default_rng(17)
    e = rand_elements(rng, "block", 300, 3)
    s0 = torch.as_tensor(rng.normal(size=6))
    dev = lambda x: x.to(cuda_device)
    eb = cs.Block2x2Elements(*[dev(x) for x in (e.a, e.b, e.c, e.d, e.u)])
    ed = block_to_dense(e)
    got = cs.parallel_affine_solve(eb, dev(s0), workers=3)
    want = cs.parallel_affine_solve(cs.DenseElements(dev(ed.J), dev(ed.u)), dev(s0))
    torch.testing.assert_close(got, want, atol=1e-10, rtol=0)


@pytest.mark.gpu
@pytest.mark.parametrize("chunk", [1, 7, 300])
def test_explicit_chunk_sizes(cuda_device, chunk):  # test_pscan.py:183-189 (chunking is the kernel's own)
    rng = np.random.default_rng(31)
    e = rand_elements(rng, "dense", 300, 2, device=cuda_device)
    s0 = torch.as_tensor(rng.normal(size=2), device=cuda_device)
    torch.testing.assert_close(cs.parallel_affine_solve(e, s0, workers=2, chunk=chunk),
                               cs.sequential_affine_solve(e, s0), atol=1e-10, rtol=0)


@pytest.mark.gpu
@pytest.mark.parametrize("variant", VARIANTS)
def test_identity_sequence_holds_state(cuda_device, variant):  # test_pscan.py:192-197
    T, D = 64, 3
    like = rand_elements(np.random.default_rng(5), variant, T, D, device=cuda_device)
    e = cs.identity_element(like)
    s0 = torch.tensor([4.0, -1.0, 0.25, 2.0, 0.5, -3.0][:like.dim], device=cuda_device, dtype=torch.float64)
    out = cs.parallel_affine_solve(e, s0, workers=2)
    assert bool((out == s0).all())


@pytest.mark.gpu
def test_allocation_accounting(cuda_device):  # test_pscan.py:206-229 (element bytes; our scratch differs)
    rng = np.random.default_rng(37)
    T, D = 4096, 5
    for variant, per in (("diag", 2 * D), ("block", 6 * D)):
        stats = {}
        e = rand_elements(rng, variant, T, D, device=cuda_device)
        cs.parallel_affine_solve(e, torch.zeros(e.dim, device=cuda_device, dtype=torch.float64), stats=stats)
        assert stats["element_bytes"] == per * T * 8
        assert stats["output_bytes"] == T * e.dim * 8
        assert stats["scratch_bytes"] < stats["element_bytes"] / 10
    stats = {}
    e = rand_elements(rng, "dense", 512, 3, device=cuda_device)
    cs.parallel_affine_solve(e, torch.zeros(3, device=cuda_device, dtype=torch.float64), stats=stats)
    assert stats["element_bytes"] == (9 + 3) * 512 * 8


@pytest.mark.gpu
def test_bad_s0_shapes_rejected(cuda_device):  # test_pscan.py:232-241
    e = cs.DiagElements(torch.ones((4, 3), device=cuda_device), torch.zeros((4, 3), device=cuda_device))
    with pytest.raises(StructuralError):
        cs.parallel_affine_solve(e, torch.zeros(2, device=cuda_device))
    z = lambda *s: torch.zeros(s, device=cuda_device)
    b = cs.Block2x2Elements(z(4, 3) + 1, z(4, 3), z(4, 3), z(4, 3) + 1, z(4, 6))
    with pytest.raises(StructuralError):
        cs.parallel_affine_solve(b, torch.zeros(3, device=cuda_device))

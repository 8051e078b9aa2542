"""The reference's test_noise.py and test_core.py restated against this package's
API (device noise tables, the TransitionSystem plugin surface, the sequential
evaluator); each test cites the reference test it mirrors."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

cs = pytest.importorskip("paper_2508_18413_b200")


def np_(t):
    return t.detach().cpu().numpy() if torch.is_tensor(t) else np.asarray(t)


def make_table(seed=7, T=100):
    layout = {"xi": cs.SlotSpec(3, "standard-normal"), "u": cs.SlotSpec(1, "uniform-0-1"),
              "g": cs.SlotSpec(2, "chi-squared", df=9.1)}
    return cs.NoiseTable(seed, layout, T)


# ---- noise (test_noise.py) ----------------------------------------------------


def test_purity_bit_identical(cuda_device):  # test_noise.py:19-25
    t = make_table()
    a = t.noise_at(3, "xi", 0)
    assert a == t.noise_at(3, "xi", 0)
    assert make_table().noise_at(3, "xi", 0) == a


def test_block_matches_scalar_access(cuda_device):  # test_noise.py:28-33
    t = make_table()
    blk = np_(t.block("xi", np.arange(10)))
    for ti in range(10):
        for k in range(3):
            assert blk[ti, k] == t.noise_at(ti, "xi", k)


def test_uniform_open_interval(cuda_device):  # test_noise.py:36-41
    u = np_(cs.NoiseTable(11, {"u": cs.SlotSpec(10, "uniform-0-1")}, T=100_000).block("u", np.arange(100_000)))
    assert u.size == 1_000_000 and np.all(u > 0.0) and np.all(u < 1.0)


def test_normal_moments(cuda_device):  # test_noise.py:44-48
    z = np_(cs.NoiseTable(5, {"xi": cs.SlotSpec(10, "standard-normal")}, T=100_000).block("xi", np.arange(100_000)))
    assert abs(z.mean()) < 0.005 and abs(z.std() - 1.0) < 0.01


def test_seed_changes_values(cuda_device):  # test_noise.py:51-54
    a = cs.NoiseTable(1, {"u": cs.SlotSpec(1, "uniform-0-1")}, T=10)
    b = cs.NoiseTable(2, {"u": cs.SlotSpec(1, "uniform-0-1")}, T=10)
    assert a.noise_at(0, "u", 0) != b.noise_at(0, "u", 0)


def test_slot_independence(cuda_device):  # test_noise.py:57-69
    lean = cs.NoiseTable(7, {"u": cs.SlotSpec(1, "uniform-0-1")}, T=50)
    fat = make_table(seed=7, T=50)
    for ti in (0, 1, 17, 49):
        assert lean.noise_at(ti, "u", 0) == fat.noise_at(ti, "u", 0)
    both = cs.NoiseTable(7, {"u": cs.SlotSpec(1, "uniform-0-1"), "u2": cs.SlotSpec(1, "uniform-0-1")}, T=50)
    assert both.noise_at(3, "u", 0) != both.noise_at(3, "u2", 0)


def test_chi_squared_moments(cuda_device):  # test_noise.py:83-88
    df = 9.1
    x = np_(cs.NoiseTable(3, {"g": cs.SlotSpec(2, "chi-squared", df=df)}, T=100_000).block("g", np.arange(100_000)))
    assert abs(x.mean() - df) < 0.05 and abs(x.var() - 2 * df) < 0.5


def test_slot_and_index_errors(cuda_device):  # test_noise.py:91-106
    t = make_table()
    with pytest.raises(cs.ConfigurationError):
        t.noise_at(0, "nope", 0)
    with pytest.raises(IndexError):
        t.noise_at(0, "xi", 3)
    with pytest.raises(IndexError):
        make_table(T=10).noise_at(11, "xi", 0)


def test_rademacher_probe_properties(cuda_device):  # test_noise.py:120-129
    z = np_(cs.rademacher_probe(9, iteration=4, ts=np.arange(5000), sample=0, dim=6))
    assert z.shape == (5000, 6)
    assert set(np.unique(z)) == {-1.0, 1.0}
    assert abs(z.mean()) < 0.02
    assert np.array_equal(z, np_(cs.rademacher_probe(9, iteration=4, ts=np.arange(5000), sample=0, dim=6)))
    assert not np.array_equal(z, np_(cs.rademacher_probe(9, 5, np.arange(5000), 0, 6)))
    assert not np.array_equal(z, np_(cs.rademacher_probe(9, 4, np.arange(5000), 1, 6)))


# ---- transition systems (test_core.py) ------------------------------------------


class AffineToy(cs.TransitionSystem):
    """s_t = a s_{t-1} + b elementwise, no noise consumed (test_core.py:14-27)."""

    def __init__(self, dim, T, a=2.0, b=1.0):
        super().__init__(dim, cs.NoiseTable(0, {}, T))
        self.a, self.b = float(a), float(b)

    def _step_batch(self, ts, s):
        return self.a * s + self.b

    def _jvp_batch(self, ts, s, v):
        return self.a * v


class ExplodeAt(cs.TransitionSystem):  # test_core.py:30-41
    def __init__(self, bad_t, T):
        super().__init__(1, cs.NoiseTable(0, {}, T))
        self.bad_t = bad_t

    def _step_batch(self, ts, s):
        out = s + 1.0
        out[ts == self.bad_t] = float("nan")
        return out

    def _jvp_batch(self, ts, s, v):
        return v


def test_affine_toy_frozen_values(cuda_device):  # test_core.py:44-49
    trace = np_(cs.sequential_evaluate(AffineToy(1, T=3), np.array([1.0])))
    assert trace.shape == (3, 1)
    np.testing.assert_array_equal(trace[:, 0], [3.0, 7.0, 15.0])


def test_identity_system_constant(cuda_device):  # test_core.py:52-56
    s0 = np.array([0.5, -2.0, 9.0])
    assert np.all(np_(cs.sequential_evaluate(AffineToy(3, T=10, a=1.0, b=0.0), s0)) == s0)


def test_diverged_error_names_step(cuda_device):  # test_core.py:59-64
    with pytest.raises(cs.ChainDivergedError) as exc:
        cs.sequential_evaluate(ExplodeAt(bad_t=3, T=10), np.zeros(1))
    assert exc.value.step == 3 and "step 3" in str(exc.value)


def test_bad_s0_shape_rejected(cuda_device):  # test_core.py:67-72
    with pytest.raises(cs.StructuralError):
        cs.sequential_evaluate(AffineToy(2, T=4), np.zeros(3))
    with pytest.raises(cs.StructuralError):
        cs.sequential_evaluate(AffineToy(2, T=4), np.zeros((2, 2)))


def test_counters_track_batched_work(cuda_device):  # test_core.py:75-82
    s = AffineToy(2, T=8)
    s.step_batch(np.arange(1, 9), np.zeros((8, 2)))
    s.jvp_batch(np.arange(1, 5), np.zeros((4, 2)), np.ones((4, 2)))
    assert s.n_step_evals == 8 and s.n_jvp_evals == 4
    s.reset_counters()
    assert s.n_step_evals == 0 and s.n_jvp_evals == 0


def test_singleton_wrappers_match_batch(cuda_device):  # test_core.py:85-94
    s = AffineToy(2, T=4, a=0.5, b=-1.0)
    x, v = np.array([2.0, 4.0]), np.array([1.0, 0.0])
    np.testing.assert_array_equal(np_(s.step(2, x)), np_(s.step_batch(np.array([2]), x[None])[0]))
    np.testing.assert_array_equal(np_(s.jvp(2, x, v)), np_(s.jvp_batch(np.array([2]), x[None], v[None])[0]))


def test_default_dense_jacobian_from_jvp(cuda_device):  # test_core.py:97-103
    s = AffineToy(3, T=4, a=1.5)
    J = np_(s.dense_jacobian_batch(np.array([1, 2]), np.random.default_rng(0).normal(size=(2, 3))))
    assert J.shape == (2, 3, 3)
    np.testing.assert_allclose(J, np.broadcast_to(1.5 * np.eye(3), (2, 3, 3)), atol=1e-15)


def test_relaxed_defaults_to_exact_for_smooth_systems(cuda_device):  # test_core.py:106-116
    s = AffineToy(2, T=4)
    ts, x, v = np.array([1]), np.ones((1, 2)), np.full((1, 2), 0.25)
    np.testing.assert_array_equal(np_(s.relaxed_step_batch(ts, x)), np_(s.step_batch(ts, x)))
    np.testing.assert_array_equal(np_(s.relaxed_jvp_batch(ts, x, v)), np_(s.jvp_batch(ts, x, v)))


def test_user_system_solves_on_the_device_engine(cuda_device):
    # a plugin system written against the TransitionSystem API runs through
    # run_deer's host-driven engine: the affine toy is solved in one dense
    # Newton iteration (test_deer.py:191-200's affine one-shot)
    s = AffineToy(2, T=300, a=0.9, b=0.1)
    r = cs.run_deer(s, np.array([1.0, -1.0]), cs.DeerConfig(mode="dense"))
    assert r.converged and r.iterations == 1
    np.testing.assert_allclose(np_(r.trace), np_(cs.sequential_evaluate(s, np.array([1.0, -1.0]))), atol=1e-12)

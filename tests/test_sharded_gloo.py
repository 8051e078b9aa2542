"""The T-sharded driver's exchange logic on CPU: 2 processes over gloo.

Per-shard compute is the oracle (test infrastructure injected through the
ShardOps interface); the driver under test -- shard bounds, halo hand-off,
carry composition over the all-gathered shard aggregates, the collective
convergence test and error agreement -- is the product code that runs over
NCCL on GPUs.  The sharded solve must reproduce the single-process oracle
run_deer: same iterations, same per-step convergence record, trace to 1e-10.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from oracle.deer import build_elements
from oracle.errors import ChainDivergedError as OChainDiverged
from paper_2508_18413_b200.errors import ChainDivergedError
from paper_2508_18413_b200.sharded import ShardOps, gather_trace, run_deer_sharded, shard_bounds


class OracleShardOps(ShardOps):
    device = torch.device("cpu")

    def __init__(self, system):
        self.s = system

    def step(self, ts, prev):
        try:
            return torch.from_numpy(self.s.step_batch(ts.numpy(), prev.numpy())), None
        except OChainDiverged as e:
            return None, int(e.step)

    def first_nonfinite_step(self, ts, arr):
        rows = ~np.all(np.isfinite(arr.numpy().reshape(arr.shape[0], -1)), axis=1)
        return int(ts[np.flatnonzero(rows)[0]]) if rows.any() else None

    def picard_fails(self, guess, f, atol, rtol):
        return 0 if O.converged(guess.numpy(), f.numpy(), atol, rtol)[0] else 1

    def elements(self, ts, guess, halo, f, cfg, iteration):
        ocfg = O.DeerConfig(mode=cfg.mode, atol=cfg.atol, rtol=cfg.rtol, hutchinson_samples=cfg.hutchinson_samples,
                            damping=cfg.damping, clip=cfg.clip, preconditioner=cfg.preconditioner)
        try:
            return build_elements(self.s, ts.numpy(), guess.numpy(), halo.numpy(), ocfg, iteration, f.numpy()), None
        except OChainDiverged as e:
            return None, int(e.step)

    def aggregate(self, el):
        acc = O.identity_element(O.scan._row(el, 0))
        for t in range(el.u.shape[0]):
            acc = O.compose(O.scan._row(el, t), acc)
        if isinstance(el, O.DiagElements):
            flat = np.concatenate([acc.j, acc.u])
        elif isinstance(el, O.Block2x2Elements):
            n = el.a.shape[-1]
            flat = np.concatenate([acc.a, acc.b, acc.c, acc.d, acc.u[:n], acc.u[n:]])
        else:
            flat = np.concatenate([acc.J.reshape(-1), acc.u])
        return torch.from_numpy(flat)

    def scan(self, el, carry):
        return torch.from_numpy(O.parallel_affine_solve(el, carry.numpy(), chunk=el.u.shape[0]))

    def bookkeeping(self, guess, nxt, atol, rtol, iteration, last_fail):
        g, x = guess.numpy(), nxt.numpy()
        gap = np.abs(x - g)
        fail = np.any(gap > atol + rtol * np.abs(x), axis=1)
        last_fail[torch.from_numpy(fail)] = iteration
        return int(fail.sum()), float(gap.max(initial=0.0))


def _system(name, T):
    if name == "hmc":
        return O.HmcKernel(O.rosenbrock(a=0.0, b=0.1, scale1=1.0, scale2=1.0), 0.5, 8, seed=0, T=T), np.zeros(2), \
            dict(mode="diag-stochastic", clip=1.0)
    if name == "mala_dense":
        return O.MalaKernel(O.gaussian([1.0, -1.0], [[1.0, 0.0], [-0.6, 1.2]]), 0.4, seed=0, T=T), np.zeros(2), \
            dict(mode="dense")
    if name == "gibbs":
        k = O.GibbsKernel(O.generate_eight_schools(), seed=0, T=T)
        return k, k.initial_state(), dict(mode="diag-stochastic", hutchinson_samples=3,
                                          preconditioner=k.recommended_preconditioner(), max_iters=400)
    if name == "leapfrog_block":
        lf = O.LeapfrogSystem(O.rosenbrock(), 0.05, T, probe_seed=4)
        return lf, np.array([0.4, -0.3, 0.6, 0.1]), dict(mode="block2x2-stochastic", max_iters=200)
    if name == "explode":
        return O.HmcKernel(O.rosenbrock(a=0.0, b=0.1, scale1=1.0, scale2=1.0), 0.5, 8, seed=0, T=T), np.zeros(2), \
            dict(mode="diag-stochastic")
    raise KeyError(name)


def _worker(rank, world, port, name, T, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2508_18413_b200.deer import DeerConfig

        sysm, s0, kw = _system(name, T)
        sysm.dtype = torch.float64
        cfg = DeerConfig(**kw)
        try:
            res = run_deer_sharded(sysm, s0, cfg, ops=OracleShardOps(sysm))
        except ChainDivergedError as e:
            q.put((rank, "diverged", e.step, e.iteration))
            return
        full = gather_trace(res, T)
        psca = gather_trace(type(res)(trace=res.per_step_converged_at[:, None].to(torch.float64),
                                      iterations=0, delta_history=None, converged=True,
                                      per_step_converged_at=None), T)
        q.put((rank, "ok", res.iterations, res.converged, full.numpy(), psca[:, 0].numpy().astype(int),
               res.delta_history, (res.lo, res.hi)))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(name, T, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, T, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    return sorted(out, key=lambda r: r[0])


def test_shard_bounds_cover_the_chain():
    for T, G in ((10, 3), (100_000, 8), (7, 7)):
        spans = [shard_bounds(T, G, r) for r in range(G)]
        assert spans[0][0] == 0 and spans[-1][1] == T
        assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))


@pytest.mark.parametrize("name,T", [("hmc", 1200), ("mala_dense", 800), ("gibbs", 600), ("leapfrog_block", 16)])
def test_sharded_matches_single_process_oracle(name, T):
    outs = _run(name, T)
    sysm, s0, kw = _system(name, T)
    ref = O.run_deer(sysm, s0, O.DeerConfig(**kw))
    for r in outs:
        assert r[1] == "ok", r
        _, _, iters, conv, full, psca, hist, _ = r
        assert iters == ref.iterations
        assert conv == ref.converged
        np.testing.assert_allclose(full, ref.trace, atol=1e-10, rtol=1e-10)
        np.testing.assert_array_equal(psca, ref.per_step_converged_at)
        np.testing.assert_allclose(hist, ref.delta_history, rtol=1e-8, atol=1e-14)
    assert outs[0][7] == (0, T // 2) and outs[1][7] == (T // 2, T)


def test_sharded_ranks_agree_on_divergence():
    # plain diag HMC on this target blows up; every rank must
    # raise the same ChainDivergedError the single-process oracle raises
    T = 1200
    sysm, s0, kw = _system("explode", T)
    try:
        O.run_deer(sysm, s0, O.DeerConfig(**kw))
        ref = None
    except OChainDiverged as e:
        ref = (e.step, e.iteration)
    outs = _run("explode", T)
    if ref is None:
        assert all(r[1] == "ok" for r in outs)
    else:
        for r in outs:
            assert r[1] == "diverged" and (r[2], r[3]) == ref

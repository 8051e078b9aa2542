"""The T-sharded driver's streamed shard path (CUDA shard ops) across two
ranks.  The pool has one GPU per box, so both ranks share cuda:0 and exchange
through a host-side gloo group: this checks the shard arithmetic (step offsets,
halo rows, carries, the stop/error agreement) with the real kernels, not
performance -- no kernel waits on another rank's kernel."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _system(name):
    import paper_2508_18413_b200 as cs

    if name == "hmc":
        m = cs.model_logp_grad_hvp(cs.rosenbrock(a=0.0, b=0.1, scale1=1.0, scale2=1.0))
        return cs.HmcKernel(m, 0.5, 8, seed=0, T=3001), np.zeros(2), cs.DeerConfig(mode="diag-stochastic", clip=1.0)
    if name == "gibbs":
        k = cs.GibbsKernel(cs.generate_eight_schools(), seed=0, T=20_001)
        return k, k.initial_state(), cs.DeerConfig(mode="diag-stochastic", hutchinson_samples=3,
                                                   preconditioner=k.recommended_preconditioner())
    if name == "mala_dense":
        k = cs.MalaKernel(cs.model_logp_grad_hvp(cs.gaussian([1.0, -1.0], [[1.0, 0.0], [-0.6, 1.2]])), 0.4,
                          seed=0, T=2001)
        return k, np.zeros(2), cs.DeerConfig(mode="dense")
    if name in ("blr_diag", "blr_dense"):  # BASELINE cfg 3's chain (reduced T): the logistic-regression builders
        X, y, _ = cs.synthetic_credit_like(seed=20250819, n=1000, dim=100)
        m = cs.model_logp_grad_hvp(cs.blr(X, y, 1.0))
        k = cs.MalaKernel(m, 0.003, seed=4, T=601 if name == "blr_diag" else 301)
        return k, np.zeros(100), cs.DeerConfig(mode="diag-stochastic" if name == "blr_diag" else "dense")
    if name == "explode":  # plain diag quasi-Newton diverges on this chain (clip=1 is what tames it)
        m = cs.model_logp_grad_hvp(cs.rosenbrock(a=0.0, b=0.1, scale1=1.0, scale2=1.0))
        return cs.HmcKernel(m, 0.5, 8, seed=0, T=3001), np.zeros(2), cs.DeerConfig(mode="diag-stochastic")
    raise KeyError(name)


def cs_errors():
    import paper_2508_18413_b200 as cs

    return cs


def _worker(rank, world, port, name, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_2508_18413_b200.sharded import gather_trace, run_deer_sharded

        forced = name.endswith("+ops")
        k, s0, cfg = _system(name[:-4] if forced else name)
        try:
            if forced:  # the general per-kernel shard ops (CUDA tensors over a gloo group)
                from paper_2508_18413_b200.sharded import CudaShardOps

                r = run_deer_sharded(k, s0, cfg, ops=CudaShardOps(k))
            else:
                r = run_deer_sharded(k, s0, cfg)
        except cs_errors().ChainDivergedError as e:
            q.put((rank, "diverged", e.step, e.iteration))
            return
        full = gather_trace(type(r)(trace=r.trace.cpu(), iterations=0, delta_history=None, converged=True,
                                    per_step_converged_at=None), k.T)
        psca = gather_trace(type(r)(trace=r.per_step_converged_at[:, None].to(torch.float64).cpu(), iterations=0,
                                    delta_history=None, converged=True, per_step_converged_at=None), k.T)
        q.put((rank, r.stats["path"], r.iterations, r.converged, full.numpy(), psca[:, 0].numpy().astype(int)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["hmc", "gibbs", "mala_dense", "blr_diag", "blr_dense", "hmc+ops", "mala_dense+ops"])
def test_two_rank_streamed_shards_match_run_deer(cuda_device, name):
    import paper_2508_18413_b200 as cs

    k, s0, cfg = _system(name.replace("+ops", ""))
    ref = cs.run_deer(k, s0, cfg)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted([q.get(timeout=600) for _ in range(2)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
    for rank, path, its, conv, full, psca in out:
        assert path == ("sharded" if name.endswith("+ops") else "sharded-streamed")
        # the sharded solve equals the reference's chunked scan with chunk = T/2,
        # so iterations agree within one and traces within the solve tolerance
        assert abs(its - ref.iterations) <= 1 and conv == ref.converged, (rank, its, ref.iterations)
        want = ref.trace.cpu().numpy()
        if its == ref.iterations:
            np.testing.assert_allclose(full, want, atol=1e-8, rtol=1e-8)
        else:  # one more or fewer update: both within the solve's own envelope
            assert np.all(np.abs(full - want) <= 1e-4 + 1e-3 * np.abs(want))


def test_two_rank_streamed_shards_agree_on_divergence(cuda_device):
    import paper_2508_18413_b200 as cs

    k, s0, cfg = _system("explode")
    with pytest.raises(cs.ChainDivergedError) as ref:
        cs.run_deer(k, s0, cfg)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, "explode", q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted([q.get(timeout=600) for _ in range(2)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
    # every rank raises the same error; its step / iteration match the
    # single-process solve up to the +-1 iteration the chunk layout allows
    assert all(o[1] == "diverged" for o in out), out
    assert out[0][2:] == out[1][2:], out
    if ref.value.step is not None:
        assert out[0][2] == ref.value.step, (out, ref.value.step)
    if ref.value.iteration is not None:
        assert abs(out[0][3] - ref.value.iteration) <= 1, (out, ref.value.iteration)

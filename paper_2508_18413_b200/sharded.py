"""T-sharded multi-GPU Newton driver (north_star (3)).

One process per GPU.  Rank g of G owns the contiguous steps
t in (lo_g, hi_g], lo_g = floor(g T / G).  Per Newton iteration:

  1. f_t on the local steps; the first local prev row is the halo
     guess[lo_g] received from rank g-1 in the previous exchange (s0 on rank 0);
  2. collective A  all-gather [first bad proposal, first non-finite f,
                   Picard fails] -> every rank takes the same branch
                   (deer.py:263-271);
  3. local elements (Jacobian estimate, preconditioner / damping / clip) and
     the local aggregate: the composed affine map of the whole shard;
  4. collective B  all-gather [aggregate | first non-finite Jacobian]: each rank
                   applies the aggregates of ranks < g to s0 in order -> its
                   carry-in (the prefix fix-up), then replays its shard;
  5. collective C  all-gather [fail rows, delta_max, last row of the new guess]
                   = the convergence all-reduce plus next iteration's halo.

The exchanged payloads are a few to a few hundred doubles, so the NCCL calls
are latency-bound.  The result equals the reference's chunked
``parallel_affine_solve`` with chunk = T/G up to f64 rounding (the carries are
applied shard by shard exactly like _scan_kernels.py:32-36).

``ShardOps`` is the per-shard compute; ``CudaShardOps`` runs it through the
CUDA C-ABI.  The driver logic itself is device-agnostic torch code, so the
multi-process exchange is exercised on CPU with gloo in tests/.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np
import torch
import torch.distributed as dist

from .errors import ChainDivergedError, StructuralError

_NO_STEP = float(2 ** 62)
_GUARD = 1e6


def shard_bounds(T: int, world: int, rank: int):
    """Rows [lo, hi) of the chain owned by ``rank`` (contiguous, balanced)."""
    return (T * rank) // world, (T * (rank + 1)) // world


def agg_width(mode: str, D: int) -> int:
    if mode == "diag-stochastic":
        return 2 * D
    if mode == "block2x2-stochastic":
        return 3 * D          # 6 x (D/2)
    return D * D + D


def apply_agg(mode: str, agg: torch.Tensor, x: torch.Tensor) -> torch.Tensor:
    """Apply a flat aggregate (see cs_scan_aggregate) to a state vector."""
    D = x.shape[0]
    if mode == "diag-stochastic":
        return agg[:D] * x + agg[D:2 * D]
    if mode == "block2x2-stochastic":
        n = D // 2
        A, B, C, E, ux, uv = (agg[k * n:(k + 1) * n] for k in range(6))
        xs, vs = x[:n], x[n:]
        return torch.cat([A * xs + B * vs + ux, C * xs + E * vs + uv])
    M = agg[:D * D].reshape(D, D)
    return M @ x + agg[D * D:D * D + D]


@dataclass
class ShardResult:
    trace: torch.Tensor                 # this rank's rows [lo, hi)
    iterations: int
    delta_history: np.ndarray
    converged: bool
    per_step_converged_at: torch.Tensor  # this rank's rows
    lo: int = 0
    hi: int = 0
    stats: dict = field(default_factory=dict)


class ShardOps:
    """Per-shard compute interface (all tensors live on ``self.device``)."""

    device: torch.device

    def step(self, ts, prev):
        """-> (f, first bad proposal step or None)."""
        raise NotImplementedError

    def first_nonfinite_step(self, ts, arr):
        raise NotImplementedError

    def picard_fails(self, guess, f, atol, rtol) -> int:
        raise NotImplementedError

    def elements(self, ts, guess, halo, f, cfg, iteration):
        """-> (elements, first non-finite Jacobian step or None)."""
        raise NotImplementedError

    def aggregate(self, elements) -> torch.Tensor:
        raise NotImplementedError

    def scan(self, elements, carry) -> torch.Tensor:
        raise NotImplementedError

    def bookkeeping(self, guess, nxt, atol, rtol, iteration, last_fail):
        """-> (fail rows, dmax); sets last_fail[row] = iteration on failing rows."""
        raise NotImplementedError


class CudaShardOps(ShardOps):
    """CUDA realisation through the C-ABI (this rank's GPU)."""

    def __init__(self, system):
        from . import _lib

        self.sys = system
        self.device = system.device
        self.lib = _lib

    def step(self, ts, prev):
        try:
            return self.sys.step_batch(ts, prev), None
        except ChainDivergedError as e:
            if e.step is None:
                raise
            return None, int(e.step)

    def first_nonfinite_step(self, ts, arr):
        from .deer import _NO_STEP as NS, _first_nonfinite

        row = _first_nonfinite(arr)
        return None if row == NS else int(ts[row])

    def picard_fails(self, guess, f, atol, rtol):
        from .deer import converged

        ok, _ = converged(guess, f, atol, rtol)
        return 0 if ok else 1

    def elements(self, ts, guess, halo, f, cfg, iteration):
        from .deer import _build_elements

        bad = []
        el = _build_elements(self.sys, ts, guess.contiguous(), halo.contiguous(), cfg, iteration, f,
                             on_bad=bad.append)
        return el, (min(bad) if bad else None)

    def aggregate(self, el):
        from .pscan import Block2x2Elements, DenseElements, DiagElements

        lib = self.lib.load()
        if isinstance(el, DiagElements):
            mode, D, arrs, width = self.lib.CS_MODE_DIAG, el.dim, (el.j, None, None, None), 2 * el.dim
            ref = el.j
        elif isinstance(el, Block2x2Elements):
            mode, D, arrs, width = self.lib.CS_MODE_BLOCK, el.a.shape[-1], (el.a, el.b, el.c, el.d), 6 * el.a.shape[-1]
            ref = el.a
        else:
            mode, D, arrs, width = self.lib.CS_MODE_DENSE, el.dim, (el.J, None, None, None), el.dim * el.dim + el.dim
            ref = el.J
        T = el.u.shape[0]
        dt = self.lib.dtype_code(ref.dtype)
        ws_bytes = lib.cs_scan_workspace_bytes(mode, dt, T, D)
        ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=ref.device)
        out = torch.empty(width, dtype=torch.float64, device=ref.device)
        ptrs = [self.lib.ptr(None if a is None else a.contiguous()) for a in arrs]
        rc = lib.cs_scan_aggregate(mode, dt, *ptrs, self.lib.ptr(el.u.contiguous()), T, D, self.lib.ptr(out),
                                   self.lib.ptr(ws), ws_bytes, self.lib.stream_ptr())
        self.lib.check(rc)
        return out

    def scan(self, el, carry):
        from .pscan import parallel_affine_solve

        return parallel_affine_solve(el, carry)

    def bookkeeping(self, guess, nxt, atol, rtol, iteration, last_fail):
        from .deer import _bookkeeping, _scratch

        return _bookkeeping(guess.contiguous(), nxt, atol, rtol, iteration, last_fail, _scratch(guess.device))


def _gather(vec: torch.Tensor, group, world, out: torch.Tensor | None = None):
    """All-gather a small vector into a (world, n) tensor on ``vec``'s device (a
    gloo group stages CUDA vectors through the host and moves the result back).
    NCCL groups gather straight into ``out`` when given (one collective, no
    list of per-rank buffers)."""
    dev = vec.device
    if dist.get_backend(group) != "nccl":  # gloo (CPU tests): host tensors, per-rank list
        vec = vec.cpu()
        res = [torch.empty_like(vec) for _ in range(world)]
        dist.all_gather(res, vec, group=group)
        return torch.stack(res).to(dev)
    if out is None:
        out = torch.empty((world, vec.numel()), dtype=vec.dtype, device=vec.device)
    dist.all_gather_into_tensor(out, vec.contiguous(), group=group)
    return out


def _streamed_shard_ok(system, cfg) -> bool:
    """Built-in systems whose element builder takes a step range (register
    kernels, Gibbs, logistic-regression MALA): the shard runs the streamed
    engine's launches."""
    if not (getattr(system, "desc", None) is not None and not cfg.full_trace
            and getattr(system, "leapfrog_mode", "sequential") != "parallel"
            and cfg.mode in ("diag-stochastic", "block2x2-stochastic", "dense")):
        return False
    from . import _lib
    from .deer import _MODE_CODE

    d = system.desc()
    c = _lib.cs_deer_config()
    c.mode = _MODE_CODE[cfg.mode]
    c.hutchinson_samples = int(cfg.hutchinson_samples)
    return bool(_lib.load().cs_system_elements_range_supported(ctypes.byref(d), ctypes.byref(c),
                                                               _lib.dtype_code(system.dtype)))


def run_deer_sharded(system, s0, cfg, ops: ShardOps | None = None, group=None, max_iters=None) -> ShardResult:
    """run_deer (deer.py:230-328) with T sharded over the process group."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    from .deer import _pre_tensor

    _pre_tensor(cfg, "cpu", system.dim)  # length check before any launch
    if ops is None and _streamed_shard_ok(system, cfg) and (cfg.window_len is None or cfg.window_len >= system.T):
        return _run_streamed_shard(system, s0, cfg, group, world, rank, max_iters)
    ops = ops or CudaShardOps(system)
    dev = ops.device
    dtype = getattr(system, "dtype", torch.float64)
    T = system.T
    D = system.dim
    lo, hi = shard_bounds(T, world, rank)
    n = hi - lo
    if n < 1:
        raise StructuralError(f"T={T} too short for {world} shards")
    if cfg.window_len is not None and cfg.window_len < T:
        raise StructuralError("sliding windows are not sharded (SURVEY.md 8e): run them per GPU")
    from .deer import default_max_iters

    max_iters = cfg.max_iters if cfg.max_iters is not None else (max_iters or default_max_iters(T))
    s0 = torch.as_tensor(s0, dtype=dtype, device=dev).reshape(D)
    ts = torch.arange(lo + 1, hi + 1, device=dev)
    guess = s0.expand(n, -1).clone()
    halo = s0.clone()
    last_fail = torch.zeros(n, dtype=torch.int32, device=dev)
    hist = []
    d0 = None
    it = 0
    done = False
    W = agg_width(cfg.mode, D)
    stats = {"path": "sharded", "world": world, "rows": (lo, hi), "collectives_per_iteration": 3}

    while True:
        prev = torch.cat([halo[None], guess[:-1]], dim=0)
        f, bad_prop = ops.step(ts, prev)
        bad_f = None if f is None else ops.first_nonfinite_step(ts, f)
        pf = 0 if (f is None or bad_f is not None) else ops.picard_fails(guess, f, cfg.atol, cfg.rtol)
        vecA = torch.tensor([_NO_STEP if bad_prop is None else bad_prop,
                             _NO_STEP if bad_f is None else bad_f, float(pf)], dtype=torch.float64, device=dev)
        gA = _gather(vecA, group, world) if dist.is_initialized() else vecA[None]
        gbp, gbf, gpf = float(gA[:, 0].min()), float(gA[:, 1].min()), float(gA[:, 2].sum())
        if gbp < _NO_STEP:
            raise ChainDivergedError(f"non-finite {getattr(system, '_what', 'proposal')} at step {int(gbp)}",
                                     step=int(gbp))
        if gbf < _NO_STEP:
            raise ChainDivergedError(f"non-finite step value at step {int(gbf)} (iteration {it + 1})",
                                     step=int(gbf), iteration=it + 1)
        if gpf == 0:
            done = True
            break
        if it >= max_iters:
            break
        el, bad_j = ops.elements(ts, guess, halo if rank > 0 else s0, f, cfg, it)
        agg = ops.aggregate(el) if bad_j is None else torch.zeros(W, dtype=torch.float64, device=dev)
        vecB = torch.cat([agg.to(torch.float64),
                          torch.tensor([_NO_STEP if bad_j is None else bad_j], dtype=torch.float64, device=dev)])
        gB = _gather(vecB, group, world) if dist.is_initialized() else vecB[None]
        gbj = float(gB[:, W].min())
        if gbj < _NO_STEP:
            raise ChainDivergedError(f"non-finite jacobian at step {int(gbj)} (iteration {it + 1})",
                                     step=int(gbj), iteration=it + 1)
        carry = s0.to(torch.float64)
        for q in range(rank):  # prefix fix-up, shard by shard (_scan_kernels.py:32-36)
            carry = apply_agg(cfg.mode, gB[q, :W], carry)
        nxt = ops.scan(el, carry.to(dtype))
        it += 1
        nfail, dmax = ops.bookkeeping(guess, nxt, cfg.atol, cfg.rtol, it, last_fail)
        vecC = torch.cat([torch.tensor([float(nfail), dmax], dtype=torch.float64, device=dev),
                          nxt[-1].to(torch.float64)])
        gC = _gather(vecC, group, world) if dist.is_initialized() else vecC[None]
        tot_fail = float(gC[:, 0].sum())
        dm = gC[:, 1]
        dmax_g = float("nan") if bool(torch.isnan(dm).any()) else float(dm.max())
        hist.append(dmax_g)
        guess = nxt
        halo = gC[rank - 1, 2:].to(dtype) if rank > 0 else s0
        if d0 is None:
            d0 = dmax_g
        if d0 > 0 and dmax_g > _GUARD * d0:
            raise ChainDivergedError(f"fixed-point iteration diverging: delta_max {dmax_g:.3e} exceeds "
                                     f"{_GUARD:.0e} x initial {d0:.3e}", iteration=it)
        if tot_fail == 0:
            done = True
            break
    return ShardResult(trace=guess, iterations=it, delta_history=np.array(hist), converged=done,
                       per_step_converged_at=last_fail + 1, lo=lo, hi=hi, stats=stats)


def _run_streamed_shard(system, s0, cfg, group, world, rank, max_iters) -> ShardResult:
    """The sharded iteration of run_deer_sharded with the streamed engine's kernels
    on this rank's steps: ONE element launch for f, the finite/Picard checks and
    the elements of steps lo+1..hi (cs_system_elements_range: noise and probes at
    the absolute step, the halo row as the state before step lo+1), the shard
    aggregate, the scan from the carry with the bookkeeping fused into its
    replay -- and the same three small all-gathers and the same error/stop order
    as the general loop above (deer.py:261-286)."""
    from . import _lib
    from .deer import _MODE_CODE, _STATS_BYTES, _parse_stats, _pre_tensor, default_max_iters

    lib = _lib.load()
    dev, dtype = system.device, system.dtype
    T, D = system.T, system.dim
    lo, hi = shard_bounds(T, world, rank)
    n = hi - lo
    if n < 1:
        raise StructuralError(f"T={T} too short for {world} shards")
    max_iters = cfg.max_iters if cfg.max_iters is not None else (max_iters or default_max_iters(T))
    dt = _lib.dtype_code(dtype)
    st = _lib.stream_ptr()
    d = system.desc()
    c = _lib.cs_deer_config()
    c.mode = _MODE_CODE[cfg.mode]
    c.atol, c.rtol = float(cfg.atol), float(cfg.rtol)
    c.max_iters = int(max_iters)
    c.hutchinson_samples = int(cfg.hutchinson_samples)
    c.damping, c.clip = float(cfg.damping), float(cfg.clip)
    pre = _pre_tensor(cfg, dev, D)
    c.preconditioner = 0 if pre is None else pre.data_ptr()
    mode = cfg.mode
    half = D // 2 if mode == "block2x2-stochastic" else D
    if mode == "diag-stochastic":
        E = [torch.empty((n, D), dtype=dtype, device=dev)]
    elif mode == "dense":
        E = [torch.empty((n, D, D), dtype=dtype, device=dev)]
    else:
        E = [torch.empty((n, half), dtype=dtype, device=dev) for _ in range(4)]
    u = torch.empty((n, D), dtype=dtype, device=dev)
    eptr = [_lib.ptr(x) for x in E] + [_lib.ptr(None)] * (4 - len(E))
    ws_bytes = lib.cs_scan_workspace_bytes(c.mode, dt, n, half)
    ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=dev)
    stats = torch.zeros(_STATS_BYTES, dtype=torch.uint8, device=dev)
    sptr = _lib.ptr(stats)
    W = agg_width(mode, D)
    agg = torch.empty(W, dtype=torch.float64, device=dev)
    s0 = torch.as_tensor(s0, dtype=dtype, device=dev).reshape(D).contiguous()
    guess = s0.expand(n, -1).clone()
    nxt = torch.empty_like(guess)
    halo = s0.clone()
    last_fail = torch.zeros(n, dtype=torch.int32, device=dev)
    hist, d0, it, done = [], None, 0, False
    use_dist = dist.is_initialized()
    stats_info = {"path": "sharded-streamed", "world": world, "rows": (lo, hi), "collectives_per_iteration": 3}
    vB = torch.empty(W + 1, dtype=torch.float64, device=dev)
    vC = torch.empty(2 + D, dtype=torch.float64, device=dev)
    oA = torch.empty((world, 4), dtype=torch.float64, device=dev)
    oB = torch.empty((world, W + 1), dtype=torch.float64, device=dev)
    oC = torch.empty((world, 2 + D), dtype=torch.float64, device=dev)
    both = torch.empty(2 * world + 4 * world, dtype=torch.float64, device=dev)
    both_h = torch.empty(both.numel(), dtype=torch.float64).pin_memory() if dev.type == "cuda" else None

    def build(it_, halo_):
        rc_ = lib.cs_system_elements_range(ctypes.byref(d), ctypes.byref(c), dt, it_, lo, n, _lib.ptr(halo_),
                                           _lib.ptr(guess), *eptr, _lib.ptr(u), sptr, st)
        _lib.check(rc_)

    def flags_dev():  # [bad_prop, bad_f, picard_fail, bad_jac] from the stats words, on the device
        i64 = stats[:24].view(torch.int64)
        return torch.cat([i64[:2].double(), stats[24:28].view(torch.int32).double(), i64[2:3].double()])

    # With a process group, one host read per iteration: the next iteration's
    # elements are built speculatively from the device-side halo while the
    # convergence exchange is in flight, and both gathered vectors come back
    # together (the speculative build is discarded when the chain stops).
    build(0, halo)
    if use_dist:
        gA = _gather(flags_dev(), group, world).cpu().numpy()
    else:
        bp, bf, bj, pc, _, _ = _parse_stats(stats)
        gA = np.array([[float(bp), float(bf), float(pc), float(bj)]])
    while True:
        gbp, gbf, gpf = float(gA[:, 0].min()), float(gA[:, 1].min()), float(gA[:, 2].sum())
        if gbp < _NO_STEP:
            raise ChainDivergedError(f"non-finite {getattr(system, '_what', 'proposal')} at step {int(gbp)}",
                                     step=int(gbp))
        if gbf < _NO_STEP:
            raise ChainDivergedError(f"non-finite step value at step {int(gbf)} (iteration {it + 1})",
                                     step=int(gbf), iteration=it + 1)
        if gpf == 0:
            done = True
            break
        if it >= max_iters:
            break
        gbj = float(gA[:, 3].min())
        if gbj < _NO_STEP:
            raise ChainDivergedError(f"non-finite jacobian at step {int(gbj)} (iteration {it + 1})",
                                     step=int(gbj), iteration=it + 1)
        if world > 1:  # shard aggregates -> carry, on the device (only lower ranks' maps are used)
            rc = lib.cs_scan_aggregate(c.mode, dt, *eptr, _lib.ptr(u), n, half, _lib.ptr(agg), _lib.ptr(ws),
                                       ws_bytes, st)
            _lib.check(rc)
            vB[:W].copy_(agg)
            vB[W].fill_(0.0)
            gB = _gather(vB, group, world, oB)
            carry = s0.to(torch.float64)
            for q in range(rank):  # prefix fix-up, shard by shard (_scan_kernels.py:32-36)
                carry = apply_agg(mode, gB[q, :W], carry)
            carry = carry.to(dtype).contiguous()
        else:
            carry = s0
        if mode == "diag-stochastic":
            rc = lib.cs_scan_diag_update(dt, eptr[0], _lib.ptr(u), _lib.ptr(carry), _lib.ptr(nxt), n, D,
                                         _lib.ptr(ws), ws_bytes, _lib.ptr(guess), c.atol, c.rtol, it + 1,
                                         _lib.ptr(last_fail), sptr, st)
        elif mode == "block2x2-stochastic":
            rc = lib.cs_scan_block_update(dt, *eptr, _lib.ptr(u), _lib.ptr(carry), _lib.ptr(nxt), n, half,
                                          _lib.ptr(ws), ws_bytes, _lib.ptr(guess), c.atol, c.rtol, it + 1,
                                          _lib.ptr(last_fail), sptr, st)
        else:
            rc = lib.cs_scan_dense(dt, eptr[0], _lib.ptr(u), _lib.ptr(carry), _lib.ptr(nxt), n, D, _lib.ptr(ws),
                                   ws_bytes, st)
            _lib.check(rc)
            base = stats.data_ptr()
            rc = lib.cs_update_bookkeeping(dt, _lib.ptr(guess), _lib.ptr(nxt), n, D, c.atol, c.rtol, it + 1,
                                           _lib.ptr(last_fail), ctypes.c_void_p(base + 28),
                                           ctypes.c_void_p(base + 32), st)
        _lib.check(rc)
        it += 1
        guess, nxt = nxt, guess
        if use_dist:
            vC[0:1].copy_(stats[28:32].view(torch.int32).double())
            vC[1:2].copy_(stats[32:40].view(torch.float64))
            vC[2:].copy_(guess[-1])
            gC_dev = _gather(vC, group, world, oC)
            if rank > 0:
                halo = gC_dev[rank - 1, 2:].to(dtype).contiguous()
            build(it, halo)  # speculative: the next iteration's elements
            gA_dev = _gather(flags_dev(), group, world, oA)
            both[:2 * world].view(world, 2).copy_(gC_dev[:, :2])
            both[2 * world:].view(world, 4).copy_(gA_dev)
            if both_h is not None:  # one pinned read for both gathered vectors
                both_h.copy_(both, non_blocking=True)
                _lib.sync_current()
                bh = both_h.numpy()
            else:
                bh = both.cpu().numpy()
            gC = bh[:2 * world].reshape(world, 2)
            gA = bh[2 * world:].reshape(world, 4)
        else:
            _, _, _, _, nfail, dmax = _parse_stats(stats)
            gC = np.array([[float(nfail), dmax]])
        tot_fail = float(gC[:, 0].sum())
        dm = gC[:, 1]
        dmax_g = float("nan") if bool(np.isnan(dm).any()) else float(dm.max())
        hist.append(dmax_g)
        if d0 is None:
            d0 = dmax_g
        if d0 > 0 and dmax_g > _GUARD * d0:
            raise ChainDivergedError(f"fixed-point iteration diverging: delta_max {dmax_g:.3e} exceeds "
                                     f"{_GUARD:.0e} x initial {d0:.3e}", iteration=it)
        if tot_fail == 0:
            done = True
            break
        if not use_dist:
            build(it, halo)
            bp, bf, bj, pc, _, _ = _parse_stats(stats)
            gA = np.array([[float(bp), float(bf), float(pc), float(bj)]])
    return ShardResult(trace=guess, iterations=it, delta_history=np.array(hist), converged=done,
                       per_step_converged_at=last_fail + 1, lo=lo, hi=hi, stats=stats_info)


def gather_trace(res: ShardResult, T: int, group=None):
    """Assemble the full (T, D) trace on every rank (tests / small T)."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world == 1:
        return res.trace
    D = res.trace.shape[1]
    pieces = []
    for r in range(world):
        lo, hi = shard_bounds(T, world, r)
        pieces.append(torch.empty((hi - lo, D), dtype=res.trace.dtype, device=res.trace.device))
    # shards can differ by one row: pad to the max and gather
    m = max(p.shape[0] for p in pieces)
    pad = torch.zeros((m, D), dtype=res.trace.dtype, device=res.trace.device)
    pad[:res.trace.shape[0]] = res.trace
    outs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(outs, pad, group=group)
    return torch.cat([o[:p.shape[0]] for o, p in zip(outs, pieces)])

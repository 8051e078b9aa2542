"""Newton fixed-point drivers for evaluating chains in parallel on B200
(mirror of chainscan/deer.py).

``run_deer`` has two realisations with identical semantics:

* fused: built-in systems (MALA / HMC on register-resident targets, Gibbs)
  without a sliding window or full trace run the WHOLE solve as one
  cooperative persistent CUDA kernel (cs_deer_solve): f_t, the Jacobian
  estimate, element formation, the scan, the convergence test and all
  bookkeeping stay on device; one host sync at the end.
* host-driven: any TransitionSystem (user systems written with torch,
  windowed solves, full traces).  Each iteration queues CUDA kernels for the
  finite checks, Picard test, Hutchinson accumulation, element formation,
  scan and bookkeeping, and reads back a few scalars to branch exactly like
  deer.py:261-319.
"""

from __future__ import annotations

import ctypes
import math
import threading
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .core import JACOBIAN_MODES, ChainDivergedError, StructuralError, TransitionSystem, as_steps
from .errors import ConfigurationError
from .noise import rademacher_probe
from .pscan import Block2x2Elements, DenseElements, DiagElements, parallel_affine_solve

__all__ = ["DeerConfig", "DeerResult", "default_max_iters", "converged", "hutchinson_diag",
           "deer_iterate", "run_deer"]

_DIVERGENCE_FACTOR = 1e6
_NO_STEP = 2 ** 63 - 1
_MODE_CODE = {"dense": _lib.CS_MODE_DENSE, "diag-stochastic": _lib.CS_MODE_DIAG,
              "block2x2-stochastic": _lib.CS_MODE_BLOCK}


def default_max_iters(T: int) -> int:
    return math.ceil(50 + 5 * T * 1e-4)


@dataclass
class DeerConfig:
    """Solver knobs (deer.py:55-93).  ``workers``/``chunk`` are accepted for API
    compatibility.  ``engine`` picks the realisation: "fused" (one persistent
    kernel), "streamed" (fused element builder + update scan per iteration),
    "host" (generic host-driven loop) or "auto"."""

    mode: str = "dense"
    atol: float = 1e-4
    rtol: float = 1e-3
    max_iters: int | None = None
    hutchinson_samples: int = 1
    damping: float = 1.0
    clip: float = math.inf
    window_len: int | None = None
    full_trace: bool = False
    preconditioner: np.ndarray | None = None
    workers: int | None = None
    chunk: int | None = None
    engine: str = "auto"

    def __post_init__(self):
        if self.mode not in JACOBIAN_MODES:
            raise ConfigurationError(f"unknown mode {self.mode!r}; expected one of {JACOBIAN_MODES}")
        if self.atol <= 0 or self.rtol < 0:
            raise ConfigurationError("need atol > 0 and rtol >= 0")
        if self.max_iters is not None and self.max_iters < 1:
            raise ConfigurationError("max_iters must be >= 1")
        if self.hutchinson_samples < 1:
            raise ConfigurationError("hutchinson_samples must be >= 1")
        if not 0.0 < self.damping <= 1.0:
            raise ConfigurationError("damping must lie in (0, 1]")
        if self.clip <= 0:
            raise ConfigurationError("clip must be positive")
        if self.window_len is not None and self.window_len < 1:
            raise ConfigurationError("window_len must be >= 1")
        if self.engine not in ("auto", "fused", "streamed", "host"):
            raise ConfigurationError(f"unknown engine {self.engine!r}")
        if self.preconditioner is not None:
            p = np.asarray(self.preconditioner.cpu() if torch.is_tensor(self.preconditioner)
                           else self.preconditioner, float)
            if p.ndim != 1 or np.any(p <= 0):
                raise ConfigurationError("preconditioner must be a positive vector")
            self.preconditioner = p


@dataclass
class DeerResult:
    trace: torch.Tensor
    iterations: int
    delta_history: np.ndarray
    converged: bool
    per_step_converged_at: torch.Tensor
    full_trace: list | None = None
    stats: dict = field(default_factory=dict)


class _Scratch:
    """Small device scalars read back once per host-driven iteration."""

    def __init__(self, device):
        self.i64 = torch.empty(1, dtype=torch.int64, device=device)
        self.u32 = torch.empty(1, dtype=torch.int32, device=device)
        self.f64 = torch.empty(1, dtype=torch.float64, device=device)


def _scratch(device):
    return _Scratch(device)


def converged(prev, next_, atol: float, rtol: float):
    """(all |next-prev| <= atol + rtol|next|, max |next-prev|) (deer.py:107-115)."""
    prev = torch.as_tensor(prev)
    next_ = torch.as_tensor(next_, dtype=prev.dtype, device=prev.device)
    if prev.shape != next_.shape:
        raise StructuralError(f"shape mismatch: {tuple(prev.shape)} vs {tuple(next_.shape)}")
    if not prev.is_cuda:
        prev, next_ = prev.cuda(), next_.cuda()
    sc = _scratch(prev.device)
    rc = _lib.load().cs_converged(_lib.dtype_code(prev.dtype), _lib.ptr(prev.contiguous()),
                                  _lib.ptr(next_.contiguous()), prev.numel(), float(atol), float(rtol),
                                  _lib.ptr(sc.u32), _lib.ptr(sc.f64), _lib.stream_ptr())
    _lib.check(rc)
    vals = torch.cat([sc.u32.to(torch.float64), sc.f64]).cpu().numpy()
    return bool(vals[0] == 0), float(vals[1])


def hutchinson_diag(jvp_batch, ts, S, n_samples: int, probe_seed: int, iteration: int):
    """mean_k z_k * (J z_k) with device Rademacher probes (deer.py:118-132)."""
    S = torch.as_tensor(S)
    est = torch.empty_like(S)
    lib = _lib.load()
    dt = _lib.dtype_code(S.dtype)
    tt = as_steps(ts, S.device)
    for k in range(n_samples):
        z = rademacher_probe(probe_seed, iteration, tt, k, S.shape[-1], dtype=S.dtype, device=S.device)
        jz = torch.as_tensor(jvp_batch(tt, S, z), dtype=S.dtype, device=S.device).contiguous()
        rc = lib.cs_hutchinson_accumulate(dt, _lib.ptr(est), _lib.ptr(z), _lib.ptr(jz), est.numel(),
                                          int(k == 0), float(n_samples) if k == n_samples - 1 else 0.0,
                                          _lib.stream_ptr())
        _lib.check(rc)
    return est


def _first_nonfinite(arr):
    arr = arr.contiguous()
    sc = _scratch(arr.device)
    width = arr[0].numel() if arr.shape[0] else 1
    rc = _lib.load().cs_first_nonfinite_row(_lib.dtype_code(arr.dtype), _lib.ptr(arr), arr.shape[0], width,
                                            _lib.ptr(sc.i64), _lib.stream_ptr())
    _lib.check(rc)
    return int(sc.i64.item())


def _first_nonfinite_into(arr, out):
    """Device-side first non-finite row (INT64_MAX if none) into out (1-elem i64)."""
    arr = arr.contiguous()
    width = arr[0].numel() if arr.shape[0] else 1
    rc = _lib.load().cs_first_nonfinite_row(_lib.dtype_code(arr.dtype), _lib.ptr(arr), arr.shape[0], width,
                                            _lib.ptr(out), _lib.stream_ptr())
    _lib.check(rc)


def _check_finite(arr, what, ts, iteration):
    row = _first_nonfinite(arr)
    if row != _NO_STEP:
        t = int(ts[row])
        raise ChainDivergedError(f"non-finite {what} at step {t} (iteration {iteration + 1})",
                                 step=t, iteration=iteration + 1)


def _pre_tensor(cfg, device, D=None):
    """The preconditioner as a (D,) f64 device vector.  The kernels read D
    entries, so the length is checked here, before any launch: length D, or
    length 1 broadcast like the reference's ``d * pre`` / ``pre[None,:]``
    products (deer.py:163-164, :177-178); block mode slices it into x and v
    halves (deer.py:192-195), which needs all D entries."""
    if cfg.preconditioner is None:
        return None
    pre = torch.as_tensor(cfg.preconditioner, dtype=torch.float64, device=device).reshape(-1)
    if D is not None and pre.shape[0] != D:
        if pre.shape[0] == 1 and cfg.mode != "block2x2-stochastic":
            return pre.expand(D).contiguous()
        raise StructuralError(f"preconditioner has length {pre.shape[0]}, the state has dimension {D}")
    return pre


def _build_elements(system, ts, guess, s0_local, cfg, iteration, f, on_bad=None, prev=None):
    """Jacobian estimate -> affine elements with preconditioner, damping and clip
    in the reference's order, u = f - Jhat prev (deer.py:157-204).

    A non-finite Jacobian raises ChainDivergedError, or, with ``on_bad`` given,
    is reported as on_bad(step) so a sharded caller can agree on it first.
    """
    lib = _lib.load()
    dt = _lib.dtype_code(guess.dtype)
    st = _lib.stream_ptr()
    if prev is None:  # the caller's prev (same tensor as step_batch saw) keeps system caches warm
        prev = torch.cat([s0_local[None], guess[:-1]], dim=0)
    f = f.to(guess.dtype).contiguous()
    T, W = guess.shape
    pre = _pre_tensor(cfg, guess.device, W)
    clip = float(cfg.clip)

    def finite_or(arr, what):
        if isinstance(on_bad, torch.Tensor):  # deferred: first bad row lands on device
            _first_nonfinite_into(arr, on_bad)
            return
        row = _first_nonfinite(arr)
        if row == _NO_STEP:
            return
        t = int(ts[row])
        if on_bad is not None:
            on_bad(t)
            return
        raise ChainDivergedError(f"non-finite {what} at step {t} (iteration {iteration + 1})",
                                 step=t, iteration=iteration + 1)

    if cfg.mode == "dense":
        Jin = torch.as_tensor(system.dense_jacobian_batch(ts, prev), dtype=guess.dtype).contiguous()
        finite_or(Jin, "jacobian")
        J = torch.empty_like(Jin)
        u = torch.empty_like(f)
        rc = lib.cs_form_dense(dt, _lib.ptr(Jin), _lib.ptr(f), _lib.ptr(s0_local), _lib.ptr(guess), T, W,
                               _lib.ptr(pre), float(cfg.damping), clip, _lib.ptr(J), _lib.ptr(u), st)
        _lib.check(rc)
        return DenseElements(J, u)
    if cfg.mode == "diag-stochastic":
        d = hutchinson_diag(system.jvp_batch, ts, prev, cfg.hutchinson_samples, system.noise.seed, iteration)
        finite_or(d, "jacobian diagonal")
        j = torch.empty_like(d)
        u = torch.empty_like(f)
        rc = lib.cs_form_diag(dt, _lib.ptr(d.contiguous()), _lib.ptr(f), _lib.ptr(s0_local), _lib.ptr(guess), T,
                              W, _lib.ptr(pre), float(cfg.damping), clip, _lib.ptr(j), _lib.ptr(u), st)
        _lib.check(rc)
        return DiagElements(j, u)
    a, b, c, dd = (torch.as_tensor(x, dtype=guess.dtype).contiguous() for x in
                   system.block_jacobian_batch(ts, prev, cfg.hutchinson_samples, iteration))
    finite_or(torch.cat([a, b, c, dd], dim=-1), "block jacobian")
    half = a.shape[-1]
    outs = [torch.empty_like(a) for _ in range(4)]
    u = torch.empty_like(f)
    rc = lib.cs_form_block(dt, _lib.ptr(a), _lib.ptr(b), _lib.ptr(c), _lib.ptr(dd), _lib.ptr(f),
                           _lib.ptr(s0_local), _lib.ptr(guess), T, half, _lib.ptr(pre), float(cfg.damping), clip,
                           *[_lib.ptr(o) for o in outs], _lib.ptr(u), st)
    _lib.check(rc)
    return Block2x2Elements(*outs, u)


def _iterate_range(system, ts, guess, s0_local, cfg, iteration, f=None, prev=None):
    """One Newton update on the steps ts seeded from s0_local (deer.py:147-208)."""
    guess = guess.contiguous()
    s0_local = s0_local.contiguous()
    if f is None:
        prev = torch.cat([s0_local[None], guess[:-1]], dim=0)
        f = system.step_batch(ts, prev)
        _check_finite(f, "step value", ts, iteration)
    elements = _build_elements(system, ts, guess, s0_local, cfg, iteration, f, prev=prev)
    return parallel_affine_solve(elements, s0_local)


def deer_iterate(system: TransitionSystem, guess, s0, cfg: DeerConfig, iteration: int = 0):
    """One full-sequence Newton update from ``guess`` (deer.py:211-218)."""
    guess = torch.as_tensor(guess, dtype=system.dtype, device=system.device)
    s0 = torch.as_tensor(s0, dtype=system.dtype, device=system.device)
    ts = torch.arange(1, guess.shape[0] + 1, device=system.device)
    return _iterate_range(system, ts, guess, s0, cfg, iteration)


def _guard(dmax, d0, iteration):
    if d0 > 0 and dmax > _DIVERGENCE_FACTOR * d0:
        raise ChainDivergedError(
            f"fixed-point iteration diverging: delta_max {dmax:.3e} exceeds "
            f"{_DIVERGENCE_FACTOR:.0e} x initial {d0:.3e}", iteration=iteration)


def _bookkeeping(guess, nxt, atol, rtol, iteration, last_fail, sc):
    T, W = guess.shape
    rc = _lib.load().cs_update_bookkeeping(_lib.dtype_code(guess.dtype), _lib.ptr(guess), _lib.ptr(nxt), T, W,
                                           float(atol), float(rtol), int(iteration), _lib.ptr(last_fail),
                                           _lib.ptr(sc.u32), _lib.ptr(sc.f64), _lib.stream_ptr())
    _lib.check(rc)
    vals = torch.cat([sc.u32.to(torch.float64), sc.f64]).cpu().numpy()
    return int(vals[0]), float(vals[1])


def _builtin_ok(system, cfg):
    """Built-in system whose elements the library builds (register kernels, or
    the GEMM-backed wide leapfrog builder), no window / full trace."""
    if getattr(system, "desc", None) is None or cfg.full_trace:
        return False
    if not getattr(system, "kernels", False):
        d = system.desc()
        if not _lib.load().cs_system_elements_supported(ctypes.byref(d), _MODE_CODE[cfg.mode],
                                                        _lib.dtype_code(system.dtype)):
            return False
    if cfg.window_len is not None and cfg.window_len < system.T:
        return False
    return getattr(system, "leapfrog_mode", "sequential") != "parallel"


def _fused_ok(system, cfg):
    if not _builtin_ok(system, cfg):
        return False
    # a property of (system kind, target, width, mode, dtype): asked once per system
    cache = system.__dict__.setdefault("_fused_support", {})
    key = (cfg.mode, system.dtype)
    if key not in cache:
        d = system.desc()
        cache[key] = bool(_lib.load().cs_deer_supported(ctypes.byref(d), _MODE_CODE[cfg.mode],
                                                        _lib.dtype_code(system.dtype)))
    return cache[key]


# persistent kernel while a thread's steps stay few (elements kept in shared
# memory); beyond that the streamed engine keeps every thread on one step
_FUSED_MAX_T = 1 << 18


def _pick_engine(system, cfg):
    if cfg.engine == "host":
        return "host"
    fused, builtin = _fused_ok(system, cfg), _builtin_ok(system, cfg)
    if cfg.engine == "fused":
        return "fused" if fused else ("streamed" if builtin else "host")
    if cfg.engine == "streamed":
        return "streamed" if builtin else "host"
    if fused and system.T <= _FUSED_MAX_T and getattr(system, "_kind", -1) != _lib.CS_SYS_GIBBS:
        return "fused"
    if builtin:
        return "streamed"
    return "host"


def _run_fused(system, s0, cfg, max_iters):
    lib = _lib.load()
    T, D = system.T, system.dim
    dev, dtype = system.device, system.dtype
    d = system.desc()
    trace = torch.empty((T, D), dtype=dtype, device=dev)
    psca = torch.empty(T, dtype=torch.int32, device=dev)
    # delta history straight into pinned host memory (UVA: the kernel's one
    # store per iteration lands on the host; no second read-back after the solve)
    hist = _pinned_hist(max_iters)
    # the solver workspace and the config record are reused across solves of
    # this system (cs_deer_solve synchronises before returning)
    key = (cfg.mode, dtype, max_iters, cfg.atol, cfg.rtol, cfg.hutchinson_samples, cfg.damping, cfg.clip,
           None if cfg.preconditioner is None else cfg.preconditioner.tobytes(), T, dev)
    cache = system.__dict__.setdefault("_fused_ws", {})
    hit = cache.get(key)
    if hit is None:
        ws_bytes = lib.cs_deer_workspace_bytes(ctypes.byref(d), _lib.dtype_code(dtype), max_iters)
        ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
        pre = _pre_tensor(cfg, dev, D)
        c = _lib.cs_deer_config()
        c.mode = _MODE_CODE[cfg.mode]
        c.atol, c.rtol = float(cfg.atol), float(cfg.rtol)
        c.max_iters = int(max_iters)
        c.hutchinson_samples = int(cfg.hutchinson_samples)
        c.damping, c.clip = float(cfg.damping), float(cfg.clip)
        c.preconditioner = 0 if pre is None else pre.data_ptr()
        cache.clear()
        hit = cache[key] = (ws, ws_bytes, pre, c)
    ws, ws_bytes, pre, c = hit
    res = _lib.cs_deer_result()
    rc = lib.cs_deer_solve(ctypes.byref(d), ctypes.byref(c), _lib.dtype_code(dtype), _lib.ptr(s0.contiguous()),
                           _lib.ptr(trace), _lib.ptr(psca), _lib.ptr(hist), _lib.ptr(ws), ws_bytes,
                           ctypes.byref(res), _lib.stream_ptr())
    it = int(res.iterations)
    # work counters as the reference would have accumulated them
    passes = it + (0 if res.stop_reason in (_lib.CS_STOP_NOFAIL,) or res.err_kind == _lib.CS_DIV_GUARD else 1)
    updates = it + (1 if res.err_kind == _lib.CS_DIV_JACOBIAN else 0)
    system.n_step_evals += T * passes
    if cfg.mode == "diag-stochastic":
        system.n_jvp_evals += T * cfg.hutchinson_samples * updates
    elif cfg.mode == "dense":
        system.n_jvp_evals += T * D * updates
    else:
        system.n_hvp_evals += T * cfg.hutchinson_samples * updates
    if rc == _lib.CS_ERR_DIVERGED:
        step = None if res.err_step < 0 else int(res.err_step)
        iteration = None if res.err_iteration < 0 else int(res.err_iteration)
        kind = {_lib.CS_DIV_PROPOSAL: f"non-finite {getattr(system, '_what', 'proposal')} at step {step}",
                _lib.CS_DIV_STEP: f"non-finite step value at step {step} (iteration {iteration})",
                _lib.CS_DIV_JACOBIAN: f"non-finite jacobian at step {step} (iteration {iteration})",
                _lib.CS_DIV_GUARD: (f"fixed-point iteration diverging: delta_max {res.guard_dmax:.3e} exceeds "
                                    f"{_DIVERGENCE_FACTOR:.0e} x initial {res.guard_d0:.3e}")}[res.err_kind]
        raise ChainDivergedError(kind, step=step, iteration=iteration)
    _lib.check(rc)
    stats = {"path": "fused", "grid_blocks": int(res.grid_blocks), "steps_per_thread": int(res.steps_per_thread),
             "kept_in_registers": bool(res.kept_in_registers), "fused_tangent": bool(res.fused_tangent),
             "launches": int(res.launches), "stop_reason": int(res.stop_reason),
             "device_ms": float(res.device_ms)}
    return DeerResult(trace=trace, iterations=it, delta_history=hist[:it].numpy().copy(),
                      converged=res.status == _lib.CS_RUN_CONVERGED, per_step_converged_at=psca,
                      full_trace=None, stats=stats)


_PINNED = threading.local()  # per-thread pinned read-back buffers (threads solve concurrently)


def _pinned(kind, n, dtype):
    d = _PINNED.__dict__.setdefault(kind, {})
    buf = d.get(n)
    if buf is None:
        buf = torch.empty(n, dtype=dtype).pin_memory()
        d[n] = buf
    return buf


def _pinned_hist(n):
    # reused across solves on this thread's stream: cs_deer_solve synchronises
    # before returning, and the result copies out of it
    return _pinned("hist", n, torch.float64)


def run_deer(system: TransitionSystem, s0, cfg: DeerConfig) -> DeerResult:
    """Drive Newton iterations to convergence or max_iters (deer.py:230-328)."""
    s0 = torch.as_tensor(s0, dtype=system.dtype, device=system.device).contiguous()
    if tuple(s0.shape) != (system.dim,):
        raise StructuralError(f"s0 must have shape ({system.dim},), got {tuple(s0.shape)}")
    T = system.T
    _pre_tensor(cfg, system.device, system.dim)  # length check before any engine runs
    max_iters = cfg.max_iters if cfg.max_iters is not None else default_max_iters(T)
    if (cfg.window_len is not None and cfg.window_len < T and cfg.engine != "host" and not cfg.full_trace
            and _window_ok(system, cfg)):
        return _run_streamed_window(system, s0, cfg, max_iters)
    engine = _pick_engine(system, cfg)
    if engine == "fused":
        return _run_fused(system, s0, cfg, max_iters)
    if engine == "streamed":
        try:
            return _run_streamed(system, s0, cfg, max_iters)
        except _NotInstantiated:
            pass
    return _run_host(system, s0, cfg, max_iters)


class _NotInstantiated(Exception):
    pass


_STATS_BYTES = 40


def _parse_stats(buf, host=None, event=None):
    # one 40-byte read-back per iteration into a reused (per-thread) pinned
    # buffer: no pageable allocation, one stream sync -- or, with `host` and
    # `event`, a copy already queued: wait for that event only (work queued
    # after it keeps the device busy while the host decides)
    if host is None:
        host = _pinned("stats", buf.numel(), torch.uint8)
        host.copy_(buf, non_blocking=True)
        _lib.sync_current()
    else:
        event.synchronize()
    raw = host.numpy().tobytes()
    bad_prop, bad_step, bad_jac = np.frombuffer(raw[:24], dtype=np.int64)
    picard, fail_rows = np.frombuffer(raw[24:32], dtype=np.uint32)
    dmax = float(np.frombuffer(raw[32:40], dtype=np.float64)[0])
    return int(bad_prop), int(bad_step), int(bad_jac), int(picard), int(fail_rows), dmax


def _run_streamed(system, s0, cfg, max_iters):
    """Per iteration: the fused element builder (f, checks, Picard, Jacobian
    estimate, elements in one pass), the scan with the bookkeeping fused into its
    replay, and ONE 40-byte read-back that decides the branch (deer.py:261-286)."""
    lib = _lib.load()
    T, D = system.T, system.dim
    dev, dtype = system.device, system.dtype
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
    if mode == "diag-stochastic":
        E = [torch.empty((T, D), dtype=dtype, device=dev)]
    elif mode == "dense":
        E = [torch.empty((T, D, D), dtype=dtype, device=dev)]
    else:
        E = [torch.empty((T, D // 2), dtype=dtype, device=dev) for _ in range(4)]
    u = torch.empty((T, D), dtype=dtype, device=dev)
    eptr = [_lib.ptr(x) for x in E] + [_lib.ptr(None)] * (4 - len(E))
    half = D // 2 if mode == "block2x2-stochastic" else D
    ws_bytes = lib.cs_scan_workspace_bytes(c.mode, dt, T, half)
    ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=dev)
    # two stats records: while the host reads iteration it's, iteration it+1's
    # elements are already being built (speculatively: they depend only on the
    # new iterate and it+1, so they are exact whenever the loop goes on)
    stats2 = [torch.zeros(_STATS_BYTES, dtype=torch.uint8, device=dev) for _ in range(2)]
    hosts = [_pinned("stats_a", _STATS_BYTES, torch.uint8), _pinned("stats_b", _STATS_BYTES, torch.uint8)]
    ready = torch.cuda.Event()
    sb = 0
    stats, sptr = stats2[0], _lib.ptr(stats2[0])
    guess = s0.expand(T, D).clone()
    nxt = torch.empty_like(guess)
    last_fail = torch.zeros(T, dtype=torch.int32, device=dev)
    backup = torch.empty_like(last_fail)
    hist, d0, it, done = [], None, 0, False
    launches = 0
    nfail, picard = 1, 1
    built = False  # this iteration's elements already queued (speculation)

    def build(it_, g_, sp_):
        rc_ = lib.cs_system_elements(ctypes.byref(d), ctypes.byref(c), dt, it_, _lib.ptr(s0), _lib.ptr(g_),
                                     *eptr, _lib.ptr(u), sp_, st)
        if rc_ == _lib.CS_ERR_CONFIG and it_ == 0:
            raise _NotInstantiated()
        _lib.check(rc_)

    while True:
        if not built:
            build(it, guess, sptr)
        launches += 2
        counted = it < max_iters
        if counted:
            backup.copy_(last_fail)
            if mode == "diag-stochastic":
                rc = lib.cs_scan_diag_update(dt, eptr[0], _lib.ptr(u), _lib.ptr(s0), _lib.ptr(nxt), T, D,
                                             _lib.ptr(ws), ws_bytes, _lib.ptr(guess), c.atol, c.rtol, it + 1,
                                             _lib.ptr(last_fail), sptr, st)
            elif mode == "block2x2-stochastic":
                rc = lib.cs_scan_block_update(dt, *eptr, _lib.ptr(u), _lib.ptr(s0), _lib.ptr(nxt), T, half,
                                              _lib.ptr(ws), ws_bytes, _lib.ptr(guess), c.atol, c.rtol, it + 1,
                                              _lib.ptr(last_fail), sptr, st)
            else:
                rc = lib.cs_scan_dense(dt, eptr[0], _lib.ptr(u), _lib.ptr(s0), _lib.ptr(nxt), T, D, _lib.ptr(ws),
                                       ws_bytes, st)
                _lib.check(rc)
                base = stats.data_ptr()
                rc = lib.cs_update_bookkeeping(dt, _lib.ptr(guess), _lib.ptr(nxt), T, D, c.atol, c.rtol, it + 1,
                                               _lib.ptr(last_fail), ctypes.c_void_p(base + 28),
                                               ctypes.c_void_p(base + 32), st)
            _lib.check(rc)
            launches += 2
        hosts[sb].copy_(stats, non_blocking=True)
        ready.record()
        built = counted  # the next iteration's elements, queued before the host decides
        if built:
            build(it + 1, nxt, _lib.ptr(stats2[sb ^ 1]))
        bad_prop, bad_step, bad_jac, picard, nfail, dmax = _parse_stats(stats, hosts[sb], ready)
        if bad_prop != _NO_STEP:
            raise ChainDivergedError(f"non-finite {getattr(system, '_what', 'proposal')} at step {bad_prop}",
                                     step=bad_prop)
        if bad_step != _NO_STEP:
            raise ChainDivergedError(f"non-finite step value at step {bad_step} (iteration {it + 1})",
                                     step=bad_step, iteration=it + 1)
        if picard == 0:
            done = True
            if counted:
                last_fail.copy_(backup)
            break
        if not counted:
            break
        if bad_jac != _NO_STEP:
            raise ChainDivergedError(f"non-finite jacobian at step {bad_jac} (iteration {it + 1})",
                                     step=bad_jac, iteration=it + 1)
        it += 1
        hist.append(dmax)
        guess, nxt = nxt, guess
        sb ^= 1
        stats, sptr = stats2[sb], _lib.ptr(stats2[sb])
        if d0 is None:
            d0 = dmax
        _guard(dmax, d0, it)
        if nfail == 0:
            done = True
            break
    nofail_stop = done and picard != 0 and nfail == 0
    system.n_step_evals += T * (it if nofail_stop else it + 1)
    if mode == "diag-stochastic":
        system.n_jvp_evals += T * cfg.hutchinson_samples * it
    elif mode == "dense":
        system.n_jvp_evals += T * D * it
    else:
        system.n_hvp_evals += T * cfg.hutchinson_samples * it
    return DeerResult(trace=guess, iterations=it, delta_history=np.array(hist), converged=done,
                      per_step_converged_at=last_fail + 1, full_trace=None,
                      stats={"path": "streamed", "launches": launches})


def _window_ok(system, cfg):
    """Built-in systems whose element builder takes a step range."""
    if getattr(system, "desc", None) is None or getattr(system, "leapfrog_mode", "sequential") == "parallel":
        return False
    cache = system.__dict__.setdefault("_range_support", {})
    key = (cfg.mode, cfg.hutchinson_samples, system.dtype)
    if key not in cache:
        d = system.desc()
        c = _lib.cs_deer_config()
        c.mode = _MODE_CODE[cfg.mode]
        c.hutchinson_samples = int(cfg.hutchinson_samples)
        cache[key] = bool(_lib.load().cs_system_elements_range_supported(ctypes.byref(d), ctypes.byref(c),
                                                                          _lib.dtype_code(system.dtype)))
    return cache[key]


def _run_streamed_window(system, s0, cfg, max_iters):
    """The sliding-window solve of deer.py:287-319 on the device: each pass
    builds f, the Picard test and the elements of the window's steps in ONE
    launch (cs_system_elements_range: noise and probes at the absolute step,
    the seed row guess[lo-1] as the state before the window), runs the update
    scan with the bookkeeping fused (stamps last_fail[lo:hi] = iteration) and
    finds the first failing step on the device; one 48-byte read decides the
    branch and the window's advance, in the reference's order."""
    lib = _lib.load()
    T, D = system.T, system.dim
    dev, dtype = system.device, system.dtype
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
    win = int(cfg.window_len)
    if mode == "diag-stochastic":
        E = [torch.empty((win, D), dtype=dtype, device=dev)]
    elif mode == "dense":
        E = [torch.empty((win, D, D), dtype=dtype, device=dev)]
    else:
        E = [torch.empty((win, D // 2), dtype=dtype, device=dev) for _ in range(4)]
    u = torch.empty((win, D), dtype=dtype, device=dev)
    eptr = [_lib.ptr(x) for x in E] + [_lib.ptr(None)] * (4 - len(E))
    half = D // 2 if mode == "block2x2-stochastic" else D
    ws_bytes = lib.cs_scan_workspace_bytes(c.mode, dt, win, half)
    ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=dev)
    buf = torch.zeros(_STATS_BYTES + 8, dtype=torch.uint8, device=dev)  # stats + first failing row
    sptr = _lib.ptr(buf)
    first_ptr = ctypes.c_void_p(buf.data_ptr() + _STATS_BYTES)
    guess = s0.expand(T, D).clone()
    nxt = torch.empty((win, D), dtype=dtype, device=dev)
    last_fail = torch.zeros(T, dtype=torch.int32, device=dev)
    backup = torch.empty(win, dtype=torch.int32, device=dev)
    host = torch.empty(_STATS_BYTES + 8, dtype=torch.uint8).pin_memory()
    hist, d0, it, w = [], None, 0, 0
    step_rows, update_rows = 0, 0  # work counters as the reference accumulates them
    while w < T:
        lo, hi = w, min(w + win, T)
        n = hi - lo
        step_rows += n
        seed = s0 if lo == 0 else guess[lo - 1]
        gw = guess[lo:hi]
        lf = last_fail[lo:hi]
        _lib.check(lib.cs_system_elements_range(ctypes.byref(d), ctypes.byref(c), dt, it, lo, n, _lib.ptr(seed),
                                                _lib.ptr(gw), *eptr, _lib.ptr(u), sptr, st))
        counted = it < max_iters
        if counted:  # the update, speculatively (discarded if the Picard test stops the window)
            backup[:n].copy_(lf)
            if mode == "diag-stochastic":
                rc = lib.cs_scan_diag_update(dt, eptr[0], _lib.ptr(u), _lib.ptr(seed), _lib.ptr(nxt), n, D,
                                             _lib.ptr(ws), ws_bytes, _lib.ptr(gw), c.atol, c.rtol, it + 1,
                                             _lib.ptr(lf), sptr, st)
            elif mode == "block2x2-stochastic":
                rc = lib.cs_scan_block_update(dt, *eptr, _lib.ptr(u), _lib.ptr(seed), _lib.ptr(nxt), n, half,
                                              _lib.ptr(ws), ws_bytes, _lib.ptr(gw), c.atol, c.rtol, it + 1,
                                              _lib.ptr(lf), sptr, st)
            else:
                rc = lib.cs_scan_dense(dt, eptr[0], _lib.ptr(u), _lib.ptr(seed), _lib.ptr(nxt), n, D, _lib.ptr(ws),
                                       ws_bytes, st)
                _lib.check(rc)
                base = buf.data_ptr()
                rc = lib.cs_update_bookkeeping(dt, _lib.ptr(gw), _lib.ptr(nxt), n, D, c.atol, c.rtol, it + 1,
                                               _lib.ptr(lf), ctypes.c_void_p(base + 28), ctypes.c_void_p(base + 32),
                                               st)
            _lib.check(rc)
            _lib.check(lib.cs_first_stamped_row(_lib.ptr(lf), n, it + 1, first_ptr, st))
        host.copy_(buf, non_blocking=True)
        _lib.sync_current()
        raw = host.numpy().tobytes()
        bad_prop, bad_step, bad_jac = np.frombuffer(raw[:24], dtype=np.int64)
        picard, nfail = np.frombuffer(raw[24:32], dtype=np.uint32)
        dmax = float(np.frombuffer(raw[32:40], dtype=np.float64)[0])
        first = int(np.frombuffer(raw[40:48], dtype=np.int64)[0])
        if bad_prop != _NO_STEP:
            raise ChainDivergedError(f"non-finite {getattr(system, '_what', 'proposal')} at step {int(bad_prop)}",
                                     step=int(bad_prop))
        if bad_step != _NO_STEP:
            raise ChainDivergedError(f"non-finite step value at step {int(bad_step)} (iteration {it + 1})",
                                     step=int(bad_step), iteration=it + 1)
        if picard == 0:  # deer.py:297-299: the window is already a fixed point
            if counted:
                lf.copy_(backup[:n])
            w = hi
            continue
        if not counted:
            break
        if bad_jac != _NO_STEP:
            raise ChainDivergedError(f"non-finite jacobian at step {int(bad_jac)} (iteration {it + 1})",
                                     step=int(bad_jac), iteration=it + 1)
        it += 1
        update_rows += n
        hist.append(dmax)
        gw.copy_(nxt[:n])
        if d0 is None:
            d0 = dmax
        _guard(dmax, d0, it)
        w = lo + first if nfail else hi
    system.n_step_evals += step_rows
    if mode == "diag-stochastic":
        system.n_jvp_evals += update_rows * cfg.hutchinson_samples
    elif mode == "dense":
        system.n_jvp_evals += update_rows * D
    else:
        system.n_hvp_evals += update_rows * cfg.hutchinson_samples
    return DeerResult(trace=guess, iterations=it, delta_history=np.array(hist), converged=w >= T,
                      per_step_converged_at=last_fail + 1, full_trace=None,
                      stats={"path": "streamed-window", "window_len": win})


def _run_host(system, s0, cfg, max_iters):
    T = system.T
    dev = system.device
    atol, rtol = cfg.atol, cfg.rtol
    guess = s0.expand(T, -1).clone()
    history: list[float] = []
    full = [] if cfg.full_trace else None
    last_fail = torch.zeros(T, dtype=torch.int32, device=dev)
    sc = _scratch(dev)
    d0 = None
    done = False
    iterations = 0

    if cfg.window_len is None or cfg.window_len >= T:
        # one device->host read per iteration: the finite check of f, the Picard
        # test, the Jacobian check and the post-update bookkeeping all land in a
        # small device buffer, and the branch below replays deer.py:263-286 in order
        ts = torch.arange(1, T + 1, device=dev)
        # 48-byte read-back: [0] bad-f row i64, [8] bad-jac row i64, [16] Picard fails u32,
        # [24] Picard dmax f64, [32] fail rows u32, [40] update dmax f64
        buf = torch.empty(48, dtype=torch.uint8, device=dev)
        base = buf.data_ptr()
        at = lambda off: ctypes.c_void_p(base + off)  # noqa: E731
        backup = torch.empty_like(last_fail)
        lib = _lib.load()
        dt = _lib.dtype_code(guess.dtype)
        while True:
            prev = torch.cat([s0[None], guess[:-1]], dim=0)
            f = system.step_batch(ts, prev).to(guess.dtype).contiguous()
            _lib.check(lib.cs_first_nonfinite_row(dt, _lib.ptr(f), T, f.shape[1], at(0), _lib.stream_ptr()))
            _lib.check(lib.cs_converged(dt, _lib.ptr(guess), _lib.ptr(f), guess.numel(), float(atol), float(rtol),
                                        at(16), at(24), _lib.stream_ptr()))
            update = iterations < max_iters
            nxt = None
            # the update is built before the Picard test is read back (one sync per
            # iteration); if the test stops the run the update is discarded, and so
            # are the jvp/hvp counts it made (deer.py:265-271 never evaluates them)
            counts = (system.n_jvp_evals, system.n_hvp_evals)
            if update:
                badj = buf[8:16].view(torch.int64)
                badj.fill_(_NO_STEP)
                el = _build_elements(system, ts, guess, s0, cfg, iterations, f, on_bad=badj, prev=prev)
                nxt = parallel_affine_solve(el, s0)
                backup.copy_(last_fail)
                _lib.check(lib.cs_update_bookkeeping(dt, _lib.ptr(guess), _lib.ptr(nxt), T, guess.shape[1],
                                                     float(atol), float(rtol), int(iterations + 1),
                                                     _lib.ptr(last_fail), at(32), at(40), _lib.stream_ptr()))
            raw = buf.cpu().numpy().tobytes()
            bad_f, bad_j = (int(v) for v in np.frombuffer(raw[0:16], dtype=np.int64))
            pic = int(np.frombuffer(raw[16:20], dtype=np.uint32)[0])
            if bad_f != _NO_STEP:
                t = int(ts[bad_f])
                raise ChainDivergedError(f"non-finite step value at step {t} (iteration {iterations + 1})",
                                         step=t, iteration=iterations + 1)
            if pic == 0:
                if update:
                    last_fail.copy_(backup)
                    system.n_jvp_evals, system.n_hvp_evals = counts
                done = True
                break
            if not update:
                break
            if bad_j != _NO_STEP:
                t = int(ts[bad_j])
                raise ChainDivergedError(f"non-finite jacobian at step {t} (iteration {iterations + 1})",
                                         step=t, iteration=iterations + 1)
            nfail = int(np.frombuffer(raw[32:36], dtype=np.uint32)[0])
            dmax = float(np.frombuffer(raw[40:48], dtype=np.float64)[0])
            iterations += 1
            history.append(dmax)
            if full is not None:
                full.append(nxt.clone())
            guess = nxt
            if d0 is None:
                d0 = dmax
            _guard(dmax, d0, iterations)
            if nfail == 0:
                done = True
                break
    else:
        win = cfg.window_len
        w = 0
        while w < T:
            lo, hi = w, min(w + win, T)
            ts = torch.arange(lo + 1, hi + 1, device=dev)
            seed_state = s0 if lo == 0 else guess[lo - 1]
            prev = torch.cat([seed_state[None], guess[lo:hi - 1]], dim=0)
            f = system.step_batch(ts, prev).to(guess.dtype)
            _check_finite(f, "step value", ts, iterations)
            ok, _ = converged(guess[lo:hi], f, atol, rtol)
            if ok:
                w = hi
                continue
            if iterations >= max_iters:
                break
            nxt = _iterate_range(system, ts, guess[lo:hi], seed_state.clone(), cfg, iterations, f=f, prev=prev)
            iterations += 1
            win_fail = torch.zeros(hi - lo, dtype=torch.int32, device=dev)
            nfail, dmax = _bookkeeping(guess[lo:hi].contiguous(), nxt, atol, rtol, 1, win_fail, sc)
            history.append(dmax)
            failmask = win_fail > 0
            last_fail[lo:hi][failmask] = iterations
            guess[lo:hi] = nxt
            if full is not None:
                full.append(guess.clone())
            if d0 is None:
                d0 = dmax
            _guard(dmax, d0, iterations)
            if nfail:
                first = int(torch.nonzero(failmask)[0, 0])
                w = lo + first
            else:
                w = hi
        done = w >= T

    return DeerResult(trace=guess, iterations=iterations, delta_history=np.array(history), converged=done,
                      per_step_converged_at=last_fail + 1, full_trace=full, stats={"path": "host"})

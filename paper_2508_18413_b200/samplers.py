"""MCMC transition kernels as deterministic transition systems on B200
(mirror of chainscan/samplers.py).

Every kernel reads its randomness from a counter-addressed NoiseTable whose
tables live in HBM.  The batched forward map, the solver-form JVP (hard gate +
sigmoid' bend), the relaxed variants, the leapfrog block estimate and the
sequential chain walk all run as fused CUDA kernels (csrc/cs_systems.cuh)
through the C-ABI; the whole-chain Newton solve over these systems runs as one
persistent kernel (deer.run_deer).  Logistic-regression MALA evaluates its data
contractions with cuBLAS GEMMs.
"""

from __future__ import annotations

import ctypes
import weakref
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .core import ChainDivergedError, StructuralError, TargetModel, TransitionSystem, as_steps
from .errors import ConfigurationError
from .noise import NoiseTable, SlotSpec, rademacher_probe

__all__ = ["MalaKernel", "mala_step", "mala_jvp", "LeapfrogSystem", "leapfrog_step",
           "leapfrog_block_jacobian", "HmcKernel", "hmc_step", "hmc_chain_system",
           "EightSchoolsHyper", "EightSchoolsData", "generate_eight_schools", "GibbsKernel",
           "gibbs_sweep", "gibbs_jvp", "CLASSIC_EFFECTS", "CLASSIC_SES"]

_NO_STEP = 2 ** 63 - 1


def _log_sigmoid(z):
    return -torch.logaddexp(torch.zeros_like(z), -z)


def _sigmoid_prime(z):
    return torch.exp(_log_sigmoid(z) + _log_sigmoid(-z))


def _noise_table(noise, slot, T, dtype, log_uniform=False):
    """(T+1, count) device table of a slot; duck-typed tables are uploaded."""
    if isinstance(noise, NoiseTable):
        return noise.table(slot, dtype, log_uniform)
    vals = torch.as_tensor(np.asarray(noise.block(slot, np.arange(T + 1))), dtype=torch.float64)
    if log_uniform:
        vals = torch.log(vals)
    return vals.to(device="cuda", dtype=dtype).contiguous()


def _first_bad(ts, values):
    rows = ~torch.isfinite(values.reshape(values.shape[0], -1)).all(dim=1)
    return int(ts[torch.nonzero(rows)[0, 0]])


class _Fused(TransitionSystem):
    """Shared plumbing for the built-in systems: descriptor + C-ABI calls."""

    _kind = -1
    _what = "proposal"

    def desc(self) -> _lib.cs_system:
        raise NotImplementedError

    def _call_step(self, ts, S, relaxed=False):
        lib = _lib.load()
        S = S.contiguous()
        out = torch.empty_like(S)
        d = self.desc()
        dt = _lib.dtype_code(self.dtype)
        if relaxed:
            rc = lib.cs_system_relaxed_step(ctypes.byref(d), dt, _lib.ptr(ts), 0, S.shape[0], _lib.ptr(S),
                                            _lib.ptr(out), _lib.stream_ptr())
            _lib.check(rc)
            return out
        bad = torch.empty(1, dtype=torch.int64, device=self.device)
        rc = lib.cs_system_step(ctypes.byref(d), dt, _lib.ptr(ts), 0, S.shape[0], _lib.ptr(S), _lib.ptr(out),
                                _lib.ptr(bad), _lib.stream_ptr())
        _lib.check(rc)
        b = int(bad.item())
        if b != _NO_STEP:
            raise ChainDivergedError(f"non-finite {self._what} at step {b}", step=b)
        return out

    def _call_jvp(self, ts, S, V, relaxed=False):
        S, V = S.contiguous(), V.contiguous()
        out = torch.empty_like(S)
        d = self.desc()
        rc = _lib.load().cs_system_jvp(ctypes.byref(d), _lib.dtype_code(self.dtype), _lib.ptr(ts), 0,
                                       S.shape[0], _lib.ptr(S), _lib.ptr(V), _lib.ptr(out), int(relaxed),
                                       _lib.stream_ptr())
        _lib.check(rc)
        return out

    # register-resident CUDA kernels when the C-ABI covers the system, else the
    # GEMM (cuBLAS) evaluation of the same arithmetic in _torch_* below
    @property
    def kernels(self) -> bool:
        if getattr(self, "_kernels", None) is None:
            d = self.desc()
            self._kernels = bool(_lib.load().cs_system_supported(ctypes.byref(d), _lib.dtype_code(self.dtype)))
        return self._kernels

    def _step_batch(self, ts, S):
        if self.kernels:
            return self._call_step(ts, S)
        return self._torch_step(ts, S, relaxed=False).to(self.dtype)

    def _jvp_batch(self, ts, S, V):
        if self.kernels:
            return self._call_jvp(ts, S, V)
        return self._torch_jvp(ts, S, V, relaxed=False).to(self.dtype)

    def relaxed_step_batch(self, ts, S):
        ts, S = as_steps(ts, self.device), self._state(S)
        if self.kernels:
            return self._call_step(ts, S, relaxed=True)
        return self._torch_step(ts, S, relaxed=True).to(self.dtype)

    def relaxed_jvp_batch(self, ts, S, V):
        ts, S, V = as_steps(ts, self.device), self._state(S), self._state(V)
        if self.kernels:
            return self._call_jvp(ts, S, V, relaxed=True)
        return self._torch_jvp(ts, S, V, relaxed=True).to(self.dtype)

    @property
    def _sequential(self):
        if self.kernels:
            return self._sequential_kernel
        # logistic-regression MALA walks on the device too (one CTA per chain)
        if self._kind == _lib.CS_SYS_MALA and getattr(self, "_blr_walk", None) is None:
            d = self.desc()
            self._blr_walk = bool(d.target.kind == _lib.CS_TARGET_BLR and d.dim <= 128 and d.target.n_data <= 4096)
        return self._sequential_kernel if getattr(self, "_blr_walk", False) else None

    def _sequential_kernel(self, s0, T):
        out = torch.empty((T, self.dim), dtype=self.dtype, device=self.device)
        bad = torch.empty(1, dtype=torch.int64, device=self.device)
        d = self.desc()
        rc = _lib.load().cs_system_sequential(ctypes.byref(d), _lib.dtype_code(self.dtype),
                                              _lib.ptr(s0.contiguous()), T, _lib.ptr(out), _lib.ptr(bad),
                                              _lib.stream_ptr())
        _lib.check(rc)
        b = int(bad.item())
        if b != _NO_STEP:
            raise ChainDivergedError(f"non-finite state at step {b}", step=b)
        return out


def _base_desc(kind, dim, model, eps, seed, T):
    d = _lib.cs_system()
    d.kind = kind
    d.dim = dim
    if model is not None:
        d.target = model.desc
    d.eps = float(eps)
    d.seed = int(seed) & 0xFFFFFFFFFFFFFFFF
    d.T = int(T)
    return d


# ---------------------------------------------------------------------------
# MALA (samplers.py:71-148)


class MalaKernel(_Fused):
    """Metropolis-adjusted Langevin transitions; noise slots "xi" (D normals)
    and "u" (one uniform)."""

    _kind = _lib.CS_SYS_MALA
    _what = "MALA proposal"

    def __init__(self, model: TargetModel, eps: float, seed: int = 0, T: int = 1,
                 noise: NoiseTable | None = None, dtype=torch.float64):
        if eps <= 0:
            raise ConfigurationError(f"MALA step size must be positive, got {eps}")
        if noise is None:
            noise = NoiseTable(seed, {"xi": SlotSpec(model.dim, "standard-normal"),
                                      "u": SlotSpec(1, "uniform-0-1")}, T)
        super().__init__(model.dim, noise, dtype)
        self.model = model
        self.eps = float(eps)

    def desc(self):
        d = _base_desc(self._kind, self.dim, self.model, self.eps, self.noise.seed, self.noise.T)
        self._xi = _noise_table(self.noise, "xi", self.noise.T, self.dtype)
        self._logu = _noise_table(self.noise, "u", self.noise.T, torch.float64, log_uniform=True)
        d.noise_vec = self._xi.data_ptr()
        d.noise_logu = self._logu.data_ptr()
        return d

    # -- GEMM evaluation (logistic regression, wide Gaussians): samplers.py:95-145 --
    # run_deer evaluates f_t(prev) and then the Hutchinson JVPs at the SAME prev;
    # the gate terms (two gradient and two log-density GEMM passes) are cached
    # for that batch so each JVP costs only its own two hvp GEMM pairs.
    def _gate(self, ts, S):
        # identity (weakref) + version: a recycled allocation never hits
        hit = getattr(self, "_gate_cache", None)
        if (hit is not None and hit[0]() is S and hit[1]() is ts and hit[2] == (S._version, ts._version)):
            return hit[3]
        out = self._gate_eval(ts, S)
        self._gate_cache = (weakref.ref(S), weakref.ref(ts), (S._version, ts._version), out)
        return out

    def _gate_eval(self, ts, S):
        eps, m = self.eps, self.model
        xi = _noise_table(self.noise, "xi", self.noise.T, torch.float64)[ts]
        S = S.to(torch.float64)
        gx = m.grad(S)
        xprop = S + eps * gx + np.sqrt(2.0 * eps) * xi
        if not bool(torch.isfinite(xprop).all()):
            b = _first_bad(ts, xprop)
            raise ChainDivergedError(f"non-finite MALA proposal at step {b}", step=b)
        gprop = m.grad(xprop)
        r_back = S - xprop - eps * gprop
        delta = (m.logp(xprop) - m.logp(S) - torch.sum(r_back * r_back, dim=-1) / (4.0 * eps)
                 + 0.5 * torch.sum(xi * xi, dim=-1))
        logu = _noise_table(self.noise, "u", self.noise.T, torch.float64, log_uniform=True)[ts, 0]
        gtilde = torch.minimum(torch.zeros_like(delta), delta) - logu
        return xprop, gx, gprop, r_back, delta, gtilde

    def _torch_step(self, ts, S, relaxed):
        xprop, *_, gtilde = self._gate(ts, S)
        S = S.to(torch.float64)
        if relaxed:
            w = torch.sigmoid(gtilde)[:, None]
            return w * xprop + (1.0 - w) * S
        return torch.where((gtilde > 0.0)[:, None], xprop, S)

    def _torch_jvp(self, ts, S, V, relaxed):
        eps, m = self.eps, self.model
        xprop, gx, gprop, r_back, delta, gtilde = self._gate(ts, S)
        S, V = S.to(torch.float64), V.to(torch.float64)
        dxprop = V + eps * m.hvp(S, V)
        dr_back = V - dxprop - eps * m.hvp(xprop, dxprop)
        ddelta = (torch.sum(gprop * dxprop, dim=-1) - torch.sum(gx * V, dim=-1)
                  - torch.sum(r_back * dr_back, dim=-1) / (2.0 * eps))
        dgate = ddelta * (delta < 0.0)
        gate = torch.sigmoid(gtilde) if relaxed else (gtilde > 0.0).to(torch.float64)
        bend = (_sigmoid_prime(gtilde) * dgate)[:, None]
        return gate[:, None] * dxprop + (1.0 - gate)[:, None] * V + (xprop - S) * bend


def mala_step(x, t, kernel: MalaKernel):
    return kernel.step(t, x)


def mala_jvp(x, v, t, kernel: MalaKernel):
    return kernel.jvp(t, x, v)


# ---------------------------------------------------------------------------
# leapfrog integrator (samplers.py:165-222)


def _checked_mass(mass, dim, device):
    if mass is None:
        return None
    m = np.asarray(mass, float)
    if m.shape != (dim,) or np.any(m <= 0):
        raise ConfigurationError("mass must be a positive vector matching the model dim")
    return torch.as_tensor(m, dtype=torch.float64, device=device)


class LeapfrogSystem(_Fused):
    """Mass-weighted leapfrog steps on the stacked [x, v] state."""

    _kind = _lib.CS_SYS_LEAPFROG

    def __init__(self, model: TargetModel, eps: float, L: int, mass=None, probe_seed: int = 0,
                 dtype=torch.float64):
        if eps <= 0 or L < 1:
            raise ConfigurationError(f"need eps > 0 and L >= 1, got eps={eps}, L={L}")
        super().__init__(2 * model.dim, NoiseTable(0, {}, L), dtype)
        self.model = model
        self.eps = float(eps)
        self.L = int(L)
        self._mass = _checked_mass(mass, model.dim, self.device)
        self.mass = np.ones(model.dim) if mass is None else np.asarray(mass, float)
        self.probe_seed = int(probe_seed)

    def desc(self):
        d = _base_desc(self._kind, self.dim, self.model, self.eps, self.noise.seed, self.L)
        d.L = self.L
        d.mass = 0 if self._mass is None else self._mass.data_ptr()
        d.probe_seed = self.probe_seed & 0xFFFFFFFFFFFFFFFF
        return d

    def _mass_t(self):
        return torch.as_tensor(self.mass, dtype=torch.float64, device=self.device)

    def _torch_step(self, ts, S, relaxed):
        h = self.model.dim
        S = S.to(torch.float64)
        x, v = S[:, :h], S[:, h:]
        xn = x + self.eps * v / self._mass_t()
        return torch.cat([xn, v + self.eps * self.model.grad(xn)], dim=-1)

    def _torch_jvp(self, ts, S, V, relaxed):
        h = self.model.dim
        S, V = S.to(torch.float64), V.to(torch.float64)
        m = self._mass_t()
        xn = S[:, :h] + self.eps * S[:, h:] / m
        dxn = V[:, :h] + self.eps * V[:, h:] / m
        return torch.cat([dxn, V[:, h:] + self.eps * self.model.hvp(xn, dxn)], dim=-1)

    def _torch_block(self, ts, S, n_samples, iteration):
        h = self.model.dim
        S = S.to(torch.float64)
        m = self._mass_t()
        xn = S[:, :h] + self.eps * S[:, h:] / m
        dhat = torch.zeros_like(xn)
        for k in range(n_samples):
            z = rademacher_probe(self.probe_seed, iteration, ts, k, h, device=self.device)
            dhat += z * self.model.hvp(xn, z)
        dhat /= n_samples
        a = torch.ones_like(dhat)
        b = (self.eps / m).expand(dhat.shape).clone()
        return a, b, self.eps * dhat, 1.0 + self.eps * self.eps * dhat / m

    def block_jacobian_batch(self, ts, S, n_samples: int, iteration: int):
        """Stochastic 2x2 block-diagonal Jacobian (samplers.py:202-222)."""
        ts = as_steps(ts, self.device)
        S = self._state(S).contiguous()
        n = S.shape[0]
        h = self.model.dim
        if not self.kernels:
            self.n_hvp_evals += int(n_samples) * n
            return tuple(x.to(self.dtype) for x in self._torch_block(ts, S, int(n_samples), int(iteration)))
        outs = [torch.empty((n, h), dtype=self.dtype, device=self.device) for _ in range(4)]
        d = self.desc()
        rc = _lib.load().cs_system_block_jacobian(ctypes.byref(d), _lib.dtype_code(self.dtype),
                                                  _lib.ptr(ts), 0, n, _lib.ptr(S), int(n_samples),
                                                  int(iteration), *[_lib.ptr(o) for o in outs],
                                                  _lib.stream_ptr())
        _lib.check(rc)
        self.n_hvp_evals += int(n_samples) * n
        return tuple(outs)


def leapfrog_step(s, kernel):
    system = kernel if isinstance(kernel, LeapfrogSystem) else kernel.leapfrog_system()
    return system.step(1, s)


def leapfrog_block_jacobian(s, kernel, n_samples: int = 1, iteration: int = 0, t: int = 1):
    system = kernel if isinstance(kernel, LeapfrogSystem) else kernel.leapfrog_system()
    a, b, c, d = system.block_jacobian_batch([t], system._state(s)[None], n_samples, iteration)
    return a[0], b[0], c[0], d[0]


# ---------------------------------------------------------------------------
# HMC (samplers.py:253-387)


class HmcKernel(_Fused):
    """HMC transitions over the chain, one proposal of L leapfrog steps each."""

    _kind = _lib.CS_SYS_HMC
    _what = "HMC trajectory"

    def __init__(self, model: TargetModel, eps: float, L: int, seed: int = 0, T: int = 1,
                 mass=None, leapfrog_mode: str = "sequential", leapfrog_cfg=None,
                 noise: NoiseTable | None = None, dtype=torch.float64):
        if eps <= 0 or L < 1:
            raise ConfigurationError(f"need eps > 0 and L >= 1, got eps={eps}, L={L}")
        if leapfrog_mode not in ("sequential", "parallel"):
            raise ConfigurationError(f"unknown leapfrog_mode {leapfrog_mode!r}")
        if noise is None:
            noise = NoiseTable(seed, {"momentum": SlotSpec(model.dim, "standard-normal"),
                                      "u": SlotSpec(1, "uniform-0-1")}, T)
        super().__init__(model.dim, noise, dtype)
        self.model = model
        self.eps = float(eps)
        self.L = int(L)
        self._mass = _checked_mass(mass, model.dim, self.device)
        self.mass = np.ones(model.dim) if mass is None else np.asarray(mass, float)
        self.leapfrog_mode = leapfrog_mode
        self.leapfrog_cfg = leapfrog_cfg
        self.fallback_events: list[tuple[int, int]] = []

    @property
    def n_leapfrog_fallbacks(self) -> int:
        return len(self.fallback_events)

    def desc(self):
        d = _base_desc(self._kind, self.dim, self.model, self.eps, self.noise.seed, self.noise.T)
        d.L = self.L
        d.mass = 0 if self._mass is None else self._mass.data_ptr()
        self._mom = _noise_table(self.noise, "momentum", self.noise.T, self.dtype)
        self._logu = _noise_table(self.noise, "u", self.noise.T, torch.float64, log_uniform=True)
        d.noise_vec = self._mom.data_ptr()
        d.noise_logu = self._logu.data_ptr()
        return d

    def leapfrog_system(self) -> LeapfrogSystem:
        return LeapfrogSystem(self.model, self.eps, self.L, None if self._mass is None else self.mass,
                              probe_seed=self.noise.seed, dtype=self.dtype)

    def _mass_t(self):
        return torch.as_tensor(self.mass, dtype=torch.float64, device=self.device)

    def _integrate_sequential(self, x, v):
        m = self._mass_t()
        for _ in range(self.L):
            x = x + self.eps * v / m
            v = v + self.eps * self.model.grad(x)
        return x, v

    def _integrate_parallel(self, ts, x, v):
        """Inner block quasi-Newton solve per proposal (samplers.py:301-320)."""
        from .deer import DeerConfig, run_deer

        cfg = self.leapfrog_cfg if self.leapfrog_cfg is not None else DeerConfig(mode="block2x2-stochastic")
        system = self.leapfrog_system()
        batched = self._integrate_parallel_batched(ts, x, v, system, cfg)
        if batched is not None:
            return batched
        xs, vs = torch.empty_like(x), torch.empty_like(v)
        h = self.model.dim
        for b in range(x.shape[0]):
            s0 = torch.cat([x[b], v[b]]).to(self.dtype)
            res = run_deer(system, s0, cfg)
            if not res.converged:
                self.fallback_events.append((int(ts[b]), res.iterations))
                xb, vb = self._integrate_sequential(x[b:b + 1], v[b:b + 1])
                xs[b], vs[b] = xb[0], vb[0]
            else:
                final = res.trace[-1].to(torch.float64)
                xs[b], vs[b] = final[:h], final[h:]
        return xs, vs

    def _integrate_parallel_batched(self, ts, x, v, system, cfg):
        """Every row's inner solve in one launch (cs_leapfrog_batch_solve: one CTA
        per proposal runs its own Newton loop); rows are then taken in order with
        the reference's semantics -- the first diverged row raises, rows that did
        not converge fall back to the sequential integrator.  None when the
        configuration needs the per-row engine (window, full trace, other modes, an
        explicitly chosen engine)."""
        from .deer import _DIVERGENCE_FACTOR, default_max_iters

        if (cfg.mode != "block2x2-stochastic" or cfg.full_trace or getattr(cfg, "engine", "auto") != "auto"
                or (cfg.window_len is not None and cfg.window_len < system.T)):
            return None
        lib = _lib.load()
        dt = _lib.dtype_code(self.dtype)
        d = system.desc()
        if not lib.cs_leapfrog_batch_supported(ctypes.byref(d), _lib.CS_MODE_BLOCK, dt):
            return None
        B = x.shape[0]
        h = self.model.dim
        s0s = torch.cat([x, v], dim=1).to(self.dtype).contiguous()
        finals = torch.empty_like(s0s)
        info = torch.empty((B, 4), dtype=torch.int32, device=self.device)
        err = torch.empty(B, dtype=torch.int64, device=self.device)
        c = _lib.cs_deer_config()
        c.mode = _lib.CS_MODE_BLOCK
        c.atol, c.rtol = float(cfg.atol), float(cfg.rtol)
        c.max_iters = int(cfg.max_iters if cfg.max_iters is not None else default_max_iters(system.T))
        c.hutchinson_samples = int(cfg.hutchinson_samples)
        c.damping, c.clip = float(cfg.damping), float(cfg.clip)
        pre = None if cfg.preconditioner is None else torch.as_tensor(cfg.preconditioner, dtype=torch.float64,
                                                                       device=self.device).contiguous()
        c.preconditioner = 0 if pre is None else pre.data_ptr()
        _lib.check(lib.cs_leapfrog_batch_solve(ctypes.byref(d), ctypes.byref(c), dt, B, _lib.ptr(s0s), _lib.ptr(finals),
                                               _lib.ptr(info), _lib.ptr(err), _lib.stream_ptr()))
        info_h, err_h = info.cpu().numpy(), err.cpu().numpy()
        ts_h = np.asarray(ts.cpu() if torch.is_tensor(ts) else ts).reshape(-1)
        xs, vs = finals[:, :h].to(torch.float64).clone(), finals[:, h:].to(torch.float64).clone()
        for b in range(B):
            status, iters, kind, eit = (int(q) for q in info_h[b])
            if status == _lib.CS_RUN_DIVERGED:
                step = None if err_h[b] < 0 else int(err_h[b])
                it = None if eit < 0 else eit
                msg = {_lib.CS_DIV_STEP: f"non-finite step value at step {step} (iteration {it})",
                       _lib.CS_DIV_JACOBIAN: f"non-finite jacobian at step {step} (iteration {it})"}.get(
                    kind, f"fixed-point iteration diverging: delta_max exceeds {_DIVERGENCE_FACTOR:.0e} x initial")
                raise ChainDivergedError(msg, step=step, iteration=it)
            if status != _lib.CS_RUN_CONVERGED:
                self.fallback_events.append((int(ts_h[b]), iters))
                xb, vb = self._integrate_sequential(x[b:b + 1], v[b:b + 1])
                xs[b], vs[b] = xb[0], vb[0]
        return xs, vs

    def _torch_step(self, ts, S, relaxed):
        xl, delta, gtilde = self._gate_torch(ts, S, parallel=False)
        S = S.to(torch.float64)
        if relaxed:
            w = torch.sigmoid(gtilde)[:, None]
            return w * xl + (1.0 - w) * S
        return torch.where((gtilde > 0.0)[:, None], xl, S)

    def _gate_torch(self, ts, S, parallel):
        eps, m = self.eps, self.model
        S64 = S.to(torch.float64)
        xi = _noise_table(self.noise, "momentum", self.noise.T, torch.float64)[ts]
        mass = self._mass_t()
        h0 = 0.5 * torch.sum(xi * xi, dim=-1) - m.logp(S64)
        v_half = torch.sqrt(mass) * xi + 0.5 * eps * m.grad(S64)
        if parallel:
            xl, v_lhalf = self._integrate_parallel(ts, S64, v_half)
        else:
            xl, v_lhalf = self._integrate_sequential(S64, v_half)
        if not bool(torch.isfinite(xl).all()):
            b = _first_bad(ts, xl)
            raise ChainDivergedError(f"non-finite HMC trajectory at step {b}", step=b)
        vl = v_lhalf - 0.5 * eps * m.grad(xl)
        hl = 0.5 * torch.sum(vl * vl / mass, dim=-1) - m.logp(xl)
        delta = h0 - hl
        logu = _noise_table(self.noise, "u", self.noise.T, torch.float64, log_uniform=True)[ts, 0]
        gtilde = torch.minimum(torch.zeros_like(delta), delta) - logu
        return xl, delta, gtilde

    def _torch_jvp(self, ts, S, V, relaxed):
        """Tangents ride the sequential integrator (samplers.py:353-381)."""
        eps, m = self.eps, self.model
        S, V = S.to(torch.float64), V.to(torch.float64)
        mass = self._mass_t()
        xi = _noise_table(self.noise, "momentum", self.noise.T, torch.float64)[ts]
        g0 = m.grad(S)
        dh0 = -torch.sum(g0 * V, dim=-1)
        h0 = 0.5 * torch.sum(xi * xi, dim=-1) - m.logp(S)
        x, v = S, torch.sqrt(mass) * xi + 0.5 * eps * g0
        dx, dv = V, 0.5 * eps * m.hvp(S, V)
        for _ in range(self.L):
            x = x + eps * v / mass
            dx = dx + eps * dv / mass
            dv = dv + eps * m.hvp(x, dx)
            v = v + eps * m.grad(x)
        gl = m.grad(x)
        vl = v - 0.5 * eps * gl
        dvl = dv - 0.5 * eps * m.hvp(x, dx)
        hl = 0.5 * torch.sum(vl * vl / mass, dim=-1) - m.logp(x)
        dhl = torch.sum(vl * dvl / mass, dim=-1) - torch.sum(gl * dx, dim=-1)
        delta, ddelta = h0 - hl, dh0 - dhl
        logu = _noise_table(self.noise, "u", self.noise.T, torch.float64, log_uniform=True)[ts, 0]
        gtilde = torch.minimum(torch.zeros_like(delta), delta) - logu
        dgate = ddelta * (delta < 0.0)
        gate = torch.sigmoid(gtilde) if relaxed else (gtilde > 0.0).to(torch.float64)
        bend = (_sigmoid_prime(gtilde) * dgate)[:, None]
        return gate[:, None] * dx + (1.0 - gate)[:, None] * V + (x - S) * bend

    def _step_batch(self, ts, S):
        if self.leapfrog_mode != "parallel":
            return super()._step_batch(ts, S)
        eps, m = self.eps, self.model
        S64 = S.to(torch.float64)
        xi = _noise_table(self.noise, "momentum", self.noise.T, torch.float64)[ts]
        mass = self._mass_t()
        h0 = 0.5 * torch.sum(xi * xi, dim=-1) - m.logp(S64)
        v_half = torch.sqrt(mass) * xi + 0.5 * eps * m.grad(S64)
        xl, v_lhalf = self._integrate_parallel(ts, S64, v_half)
        if not bool(torch.isfinite(xl).all()):
            b = _first_bad(ts, xl)
            raise ChainDivergedError(f"non-finite HMC trajectory at step {b}", step=b)
        vl = v_lhalf - 0.5 * eps * m.grad(xl)
        hl = 0.5 * torch.sum(vl * vl / mass, dim=-1) - m.logp(xl)
        delta = h0 - hl
        logu = _noise_table(self.noise, "u", self.noise.T, torch.float64, log_uniform=True)[ts, 0]
        gtilde = torch.minimum(torch.zeros_like(delta), delta) - logu
        return torch.where((gtilde > 0.0)[:, None], xl, S64).to(self.dtype)

    @property
    def _sequential(self):
        return self._sequential_kernel if (self.kernels and self.leapfrog_mode != "parallel") else None


def hmc_step(x, t, kernel: HmcKernel, leapfrog_mode: str | None = None):
    if leapfrog_mode is None or leapfrog_mode == kernel.leapfrog_mode:
        return kernel.step(t, x)
    swapped = HmcKernel(kernel.model, kernel.eps, kernel.L,
                        mass=None if kernel._mass is None else kernel.mass,
                        leapfrog_mode=leapfrog_mode, leapfrog_cfg=kernel.leapfrog_cfg,
                        noise=kernel.noise, dtype=kernel.dtype)
    out = swapped.step(t, x)
    kernel.fallback_events.extend(swapped.fallback_events)
    return out


def hmc_chain_system(model: TargetModel, eps: float, L: int, seed: int = 0, T: int = 1, mass=None,
                     leapfrog_mode: str = "sequential", leapfrog_cfg=None) -> HmcKernel:
    return HmcKernel(model, eps, L, seed=seed, T=T, mass=mass, leapfrog_mode=leapfrog_mode,
                     leapfrog_cfg=leapfrog_cfg)


# ---------------------------------------------------------------------------
# eight schools Gibbs (samplers.py:416-668)


@dataclass(frozen=True)
class EightSchoolsHyper:
    nu0: float = 0.1
    tau0_sq: float = 100.0
    mu0: float = 0.0
    kappa0: float = 0.1
    alpha0: float = 0.1
    sigma0_sq: float = 10.0


class EightSchoolsData:
    """Per-school observations plus cached sufficient statistics (samplers.py:428-438)."""

    def __init__(self, x):
        x = np.asarray(x, float)
        if x.ndim != 2:
            raise ConfigurationError(f"observations must be (schools, n), got {x.shape}")
        self.x = x
        self.n_schools, self.n_per_school = x.shape
        self.xbar = x.mean(axis=1)
        self.ss = np.sum((x - self.xbar[:, None]) ** 2, axis=1)


CLASSIC_EFFECTS = (28.0, 8.0, -3.0, 7.0, -1.0, 1.0, 18.0, 12.0)
CLASSIC_SES = (15.0, 10.0, 16.0, 11.0, 9.0, 11.0, 10.0, 18.0)


def generate_eight_schools(seed: int = 11, n_per_school: int = 20) -> EightSchoolsData:
    """Raw scores behind the classic table, means/SEs matched exactly (samplers.py:445-461)."""
    table = NoiseTable(seed, {"z": SlotSpec(n_per_school, "standard-normal")}, T=len(CLASSIC_EFFECTS))
    z_all = table.fill("z", 1, len(CLASSIC_EFFECTS)).cpu().numpy()
    rows = []
    for s, (effect, se) in enumerate(zip(CLASSIC_EFFECTS, CLASSIC_SES)):
        z = z_all[s]
        z = z - z.mean()
        z = z / z.std(ddof=1)
        rows.append(effect + z * se * np.sqrt(n_per_school))
    return EightSchoolsData(np.array(rows))


class GibbsKernel(_Fused):
    """One systematic-scan sweep of the eight-schools hierarchy (tau^2, mu,
    theta_1..S, sigma^2_1..S), reparameterised onto fixed noise."""

    _kind = _lib.CS_SYS_GIBBS
    VARIANCE_FLOOR = 1e-8

    def __init__(self, data: EightSchoolsData, hyper: EightSchoolsHyper | None = None, seed: int = 0,
                 T: int = 1, dtype=torch.float64):
        hyper = hyper or EightSchoolsHyper()
        S = data.n_schools
        layout = {
            "g_tau": SlotSpec(1, "chi-squared", df=hyper.nu0 + S + 1),
            "xi_mu": SlotSpec(1, "standard-normal"),
            "xi_theta": SlotSpec(S, "standard-normal"),
            "g_sigma": SlotSpec(S, "chi-squared", df=hyper.alpha0 + data.n_per_school),
            "g_tau_prior": SlotSpec(1, "chi-squared", df=hyper.nu0),
            "xi_mu_prior": SlotSpec(1, "standard-normal"),
            "xi_theta_prior": SlotSpec(S, "standard-normal"),
            "g_sigma_prior": SlotSpec(S, "chi-squared", df=hyper.alpha0),
        }
        super().__init__(2 * S + 2, NoiseTable(seed, layout, T), dtype)
        self.data = data
        self.hyper = hyper
        self.S = S
        h = hyper
        prm = np.concatenate([[h.nu0, h.tau0_sq, h.mu0, h.kappa0, h.alpha0, h.sigma0_sq, S,
                               data.n_per_school], data.xbar, data.ss])
        self._prm = torch.as_tensor(prm, dtype=torch.float64, device=self.device)

    def desc(self):
        d = _base_desc(self._kind, self.dim, None, 0.0, self.noise.seed, self.noise.T)
        self._tabs = [_noise_table(self.noise, s, self.noise.T, self.dtype)
                      for s in ("g_tau", "xi_mu", "xi_theta", "g_sigma")]
        d.g_tau, d.xi_mu, d.xi_theta, d.g_sigma = [t.data_ptr() for t in self._tabs]
        d.gibbs = self._prm.data_ptr()
        return d

    def unpack(self, state):
        S = self.S
        state = torch.as_tensor(state)
        return state[..., 0], state[..., 1], state[..., 2:2 + S], state[..., 2 + S:]

    def pack(self, tau2, mu, theta, sig2):
        return torch.cat([tau2[..., None], mu[..., None], theta, sig2], dim=-1)

    def recommended_preconditioner(self):
        """1e-12 on tau^2 and every sigma^2 (samplers.py:510-523)."""
        pre = np.ones(self.dim)
        pre[0] = 1e-12
        pre[2 + self.S:] = 1e-12
        return pre

    def initial_state(self):
        """Prior draw at t=0 refined by one sweep step(0, .) (samplers.py:631-641)."""
        h = self.hyper
        nz = self.noise
        g_tau0 = nz.fill("g_tau_prior", 0, 1)[0, 0]
        tau2 = h.nu0 * h.tau0_sq / g_tau0
        mu = h.mu0 + torch.sqrt(tau2 / h.kappa0) * nz.fill("xi_mu_prior", 0, 1)[0, 0]
        theta = mu + torch.sqrt(tau2) * nz.fill("xi_theta_prior", 0, 1)[0]
        sig2 = h.alpha0 * h.sigma0_sq / nz.fill("g_sigma_prior", 0, 1)[0]
        prior = self.pack(tau2.reshape(()), mu.reshape(()), theta, sig2)
        return self.step(0, prior)

    def conditional_parameters(self, state):
        """Full-conditional parameters at a fixed joint state (samplers.py:643-668)."""
        h, d = self.hyper, self.data
        S = self.S
        n = d.n_per_school
        tau2, mu, theta, sig2 = (torch.as_tensor(v, dtype=torch.float64) for v in self.unpack(
            torch.as_tensor(state, dtype=torch.float64)))
        xbar = torch.as_tensor(d.xbar, dtype=torch.float64, device=theta.device)
        ss = torch.as_tensor(d.ss, dtype=torch.float64, device=theta.device)
        df_tau = h.nu0 + S + 1
        q_tau = h.nu0 * h.tau0_sq + h.kappa0 * (mu - h.mu0) ** 2 + torch.sum((theta - mu[..., None]) ** 2, dim=-1)
        kS = h.kappa0 + S
        prec = 1.0 / tau2[..., None] + n / sig2
        df_sig = h.alpha0 + n
        return {
            "tau2": (df_tau, q_tau / df_tau),
            "mu": ((h.kappa0 * h.mu0 + theta.sum(dim=-1)) / kS, tau2 / kS),
            "theta": ((mu[..., None] / tau2[..., None] + n * xbar / sig2) / prec, 1.0 / prec),
            "sigma2": (df_sig, (h.alpha0 * h.sigma0_sq + ss + n * (xbar - theta) ** 2) / df_sig),
        }


def gibbs_sweep(state, t, kernel: GibbsKernel):
    return kernel.step(t, state)


def gibbs_jvp(state, v, t, kernel: GibbsKernel):
    return kernel.jvp(t, state, v)

"""Transition systems f_t and their Jacobian access (TEST INFRASTRUCTURE ONLY).

Reference: ``chainscan/core.py`` (TransitionSystem 61-160, sequential_evaluate
163-184) and ``chainscan/samplers.py`` (MALA 71-148, LeapfrogSystem 165-222,
HmcKernel 253-387, eight-schools data 416-461, GibbsKernel 464-668).
Arithmetic is written in the same operation order as the reference so f64
traces agree to rounding.
"""

from __future__ import annotations

import numpy as np
from scipy.special import expit

from .errors import ChainDivergedError, ConfigurationError, StructuralError
from .rng import NoiseTable, SlotSpec, rademacher_probe


def _logsig(z):
    return -np.logaddexp(0.0, -z)


def sigmoid_prime(z):
    """sigma(z) sigma(-z) in the saturation-safe log form (samplers.py:53-59)."""
    return np.exp(_logsig(z) + _logsig(-z))


def _first_bad(ts, arr):
    rows = ~np.all(np.isfinite(arr.reshape(arr.shape[0], -1)), axis=1)
    return int(np.asarray(ts)[np.flatnonzero(rows)[0]])


class System:
    """Batched f_t / jvp with work counters (core.py:61-160)."""

    def __init__(self, dim, noise=None):
        self.dim = int(dim)
        self.noise = noise
        self.n_step_evals = 0
        self.n_jvp_evals = 0
        self.n_hvp_evals = 0

    @property
    def T(self):
        if self.noise is None:
            raise ConfigurationError("system has no noise table")
        return self.noise.T

    def reset_counters(self):
        self.n_step_evals = self.n_jvp_evals = self.n_hvp_evals = 0

    def step(self, t, s):
        return self.step_batch(np.array([t]), np.asarray(s, dtype=np.float64)[None])[0]

    def step_batch(self, ts, S):
        ts = np.asarray(ts)
        self.n_step_evals += len(ts)
        return self._step_batch(ts, np.asarray(S, dtype=np.float64))

    def jvp_batch(self, ts, S, V):
        ts = np.asarray(ts)
        self.n_jvp_evals += len(ts)
        return self._jvp_batch(ts, np.asarray(S, dtype=np.float64), np.asarray(V, dtype=np.float64))

    def dense_jacobian_batch(self, ts, S):
        """Column d = jvp with the unit vector e_d (core.py:125-134)."""
        S = np.asarray(S, dtype=np.float64)
        n, D = S.shape
        J = np.empty((n, D, D))
        eye = np.eye(D)
        for d in range(D):
            J[:, :, d] = self.jvp_batch(ts, S, np.broadcast_to(eye[d], (n, D)))
        return J

    def block_jacobian_batch(self, ts, S, n_samples, iteration):
        raise ConfigurationError(f"{type(self).__name__} has no block2x2 estimate")


def sequential_evaluate(system, s0, T=None):
    """Ground-truth trace, one singleton batch per step (core.py:163-184)."""
    s = np.asarray(s0, dtype=np.float64)
    if s.ndim != 1 or s.shape[0] != system.dim:
        raise StructuralError("s0 shape")
    T = system.T if T is None else T
    out = np.empty((T, system.dim))
    for t in range(1, T + 1):
        s = system.step(t, s)
        if not np.all(np.isfinite(s)):
            raise ChainDivergedError(f"non-finite state at step {t}", step=t)
        out[t - 1] = s
    return out


# ---------------------------------------------------------------------------
# MALA (samplers.py:71-148)


class MalaKernel(System):
    def __init__(self, model, eps, seed=0, T=1, noise=None):
        if eps <= 0:
            raise ConfigurationError("eps must be positive")
        if noise is None:
            noise = NoiseTable(seed, {"xi": SlotSpec(model.dim, "standard-normal"),
                                      "u": SlotSpec(1, "uniform-0-1")}, T)
        super().__init__(model.dim, noise)
        self.model = model
        self.eps = float(eps)

    def gate_terms(self, ts, S):
        m, eps = self.model, self.eps
        xi = self.noise.block("xi", ts)
        g0 = m.grad(S)
        prop = S + eps * g0 + np.sqrt(2.0 * eps) * xi
        if not np.all(np.isfinite(prop)):
            step = _first_bad(ts, prop)
            raise ChainDivergedError(f"non-finite MALA proposal at step {step}", step=step)
        g1 = m.grad(prop)
        back = S - prop - eps * g1
        delta = (m.logp(prop) - m.logp(S) - np.sum(back * back, axis=-1) / (4.0 * eps)
                 + 0.5 * np.sum(xi * xi, axis=-1))
        margin = np.minimum(0.0, delta) - np.log(self.noise.block("u", ts)[:, 0])
        return prop, g0, g1, back, delta, margin

    def _step_batch(self, ts, S):
        prop, *_, margin = self.gate_terms(ts, S)
        return np.where((margin > 0.0)[:, None], prop, S)

    def relaxed_step_batch(self, ts, S):
        prop, *_, margin = self.gate_terms(ts, np.asarray(S, dtype=np.float64))
        w = expit(margin)[:, None]
        return w * prop + (1.0 - w) * S

    def _tangent(self, ts, S, V, hard):
        m, eps = self.model, self.eps
        prop, g0, g1, back, delta, margin = self.gate_terms(ts, S)
        dprop = V + eps * m.hvp(S, V)
        dback = V - dprop - eps * m.hvp(prop, dprop)
        ddelta = (np.sum(g1 * dprop, axis=-1) - np.sum(g0 * V, axis=-1)
                  - np.sum(back * dback, axis=-1) / (2.0 * eps))
        gate = (margin > 0.0).astype(np.float64) if hard else expit(margin)
        bend = (sigmoid_prime(margin) * (ddelta * (delta < 0.0)))[:, None]
        return gate[:, None] * dprop + (1.0 - gate)[:, None] * V + (prop - S) * bend

    def _jvp_batch(self, ts, S, V):
        return self._tangent(ts, S, V, True)

    def relaxed_jvp_batch(self, ts, S, V):
        return self._tangent(np.asarray(ts), np.asarray(S, dtype=np.float64),
                             np.asarray(V, dtype=np.float64), False)


# ---------------------------------------------------------------------------
# leapfrog + HMC (samplers.py:165-387)


def _mass(mass, dim):
    if mass is None:
        return np.ones(dim)
    mass = np.asarray(mass, dtype=np.float64)
    if mass.shape != (dim,) or np.any(mass <= 0):
        raise ConfigurationError("mass must be a positive vector")
    return mass


class LeapfrogSystem(System):
    """State [x, v]; x' = x + eps v/m, v' = v + eps grad(x')."""

    def __init__(self, model, eps, L, mass=None, probe_seed=0):
        if eps <= 0 or L < 1:
            raise ConfigurationError("need eps > 0 and L >= 1")
        super().__init__(2 * model.dim, NoiseTable(0, {}, L))
        self.model, self.eps, self.L = model, float(eps), int(L)
        self.mass = _mass(mass, model.dim)
        self.probe_seed = probe_seed

    def _step_batch(self, ts, S):
        n = self.model.dim
        x, v = S[..., :n], S[..., n:]
        xn = x + self.eps * v / self.mass
        return np.concatenate([xn, v + self.eps * self.model.grad(xn)], axis=-1)

    def _jvp_batch(self, ts, S, V):
        n = self.model.dim
        x, v, dx, dv = S[..., :n], S[..., n:], V[..., :n], V[..., n:]
        xn = x + self.eps * v / self.mass
        dxn = dx + self.eps * dv / self.mass
        return np.concatenate([dxn, dv + self.eps * self.model.hvp(xn, dxn)], axis=-1)

    def block_jacobian_batch(self, ts, S, n_samples, iteration):
        """a=1, b=eps/m, c=eps dhat, d=1+eps^2 dhat/m (samplers.py:202-222)."""
        S = np.asarray(S, dtype=np.float64)
        n = self.model.dim
        x, v = S[..., :n], S[..., n:]
        xn = x + self.eps * v / self.mass
        dhat = np.zeros_like(x)
        for k in range(n_samples):
            z = rademacher_probe(self.probe_seed, iteration, np.asarray(ts), k, n)
            dhat += z * self.model.hvp(xn, z)
        dhat /= n_samples
        self.n_hvp_evals += n_samples * len(np.asarray(ts))
        a = np.ones_like(dhat)
        b = np.broadcast_to(self.eps / self.mass, dhat.shape).copy()
        return a, b, self.eps * dhat, 1.0 + self.eps * self.eps * dhat / self.mass


class HmcKernel(System):
    def __init__(self, model, eps, L, seed=0, T=1, mass=None, leapfrog_mode="sequential",
                 leapfrog_cfg=None, noise=None):
        if eps <= 0 or L < 1:
            raise ConfigurationError("need eps > 0 and L >= 1")
        if leapfrog_mode not in ("sequential", "parallel"):
            raise ConfigurationError("unknown leapfrog_mode")
        if noise is None:
            noise = NoiseTable(seed, {"momentum": SlotSpec(model.dim, "standard-normal"),
                                      "u": SlotSpec(1, "uniform-0-1")}, T)
        super().__init__(model.dim, noise)
        self.model, self.eps, self.L = model, float(eps), int(L)
        self.mass = _mass(mass, model.dim)
        self.leapfrog_mode = leapfrog_mode
        self.leapfrog_cfg = leapfrog_cfg
        self.fallback_events = []

    def leapfrog_system(self):
        return LeapfrogSystem(self.model, self.eps, self.L, self.mass, probe_seed=self.noise.seed)

    def _seq_traj(self, x, v):
        for _ in range(self.L):
            x = x + self.eps * v / self.mass
            v = v + self.eps * self.model.grad(x)
        return x, v

    def _par_traj(self, ts, x, v):
        from .deer import DeerConfig, run_deer

        cfg = self.leapfrog_cfg or DeerConfig(mode="block2x2-stochastic")
        lf = self.leapfrog_system()
        xs, vs = np.empty_like(x), np.empty_like(v)
        n = self.model.dim
        for row in range(x.shape[0]):
            res = run_deer(lf, np.concatenate([x[row], v[row]]), cfg)
            if not res.converged:
                self.fallback_events.append((int(np.asarray(ts)[row]), res.iterations))
                xr, vr = self._seq_traj(x[row:row + 1], v[row:row + 1])
                xs[row], vs[row] = xr[0], vr[0]
            else:
                xs[row], vs[row] = res.trace[-1][:n], res.trace[-1][n:]
        return xs, vs

    def gate_terms(self, ts, S):
        m, eps = self.model, self.eps
        xi = self.noise.block("momentum", ts)
        h0 = 0.5 * np.sum(xi * xi, axis=-1) - m.logp(S)
        vh = np.sqrt(self.mass) * xi + 0.5 * eps * m.grad(S)
        if self.leapfrog_mode == "parallel":
            xl, vlh = self._par_traj(ts, S, vh)
        else:
            xl, vlh = self._seq_traj(S, vh)
        if not np.all(np.isfinite(xl)):
            step = _first_bad(ts, xl)
            raise ChainDivergedError(f"non-finite HMC trajectory at step {step}", step=step)
        vl = vlh - 0.5 * eps * m.grad(xl)
        delta = h0 - (0.5 * np.sum(vl * vl / self.mass, axis=-1) - m.logp(xl))
        margin = np.minimum(0.0, delta) - np.log(self.noise.block("u", ts)[:, 0])
        return xl, delta, margin

    def _step_batch(self, ts, S):
        xl, _, margin = self.gate_terms(ts, S)
        return np.where((margin > 0.0)[:, None], xl, S)

    def relaxed_step_batch(self, ts, S):
        S = np.asarray(S, dtype=np.float64)
        xl, _, margin = self.gate_terms(ts, S)
        w = expit(margin)[:, None]
        return w * xl + (1.0 - w) * S

    def _tangent(self, ts, S, V, hard):
        m, eps, mass = self.model, self.eps, self.mass
        xi = self.noise.block("momentum", ts)
        g0 = m.grad(S)
        dh0 = -np.sum(g0 * V, axis=-1)
        h0 = 0.5 * np.sum(xi * xi, axis=-1) - m.logp(S)
        x, v = S, np.sqrt(mass) * xi + 0.5 * eps * g0
        dx, dv = V, 0.5 * eps * m.hvp(S, V)
        for _ in range(self.L):
            x = x + eps * v / mass
            dx = dx + eps * dv / mass
            dv = dv + eps * m.hvp(x, dx)
            v = v + eps * m.grad(x)
        gl = m.grad(x)
        vl = v - 0.5 * eps * gl
        dvl = dv - 0.5 * eps * m.hvp(x, dx)
        hl = 0.5 * np.sum(vl * vl / mass, axis=-1) - m.logp(x)
        dhl = np.sum(vl * dvl / mass, axis=-1) - np.sum(gl * dx, axis=-1)
        delta, ddelta = h0 - hl, dh0 - dhl
        margin = np.minimum(0.0, delta) - np.log(self.noise.block("u", ts)[:, 0])
        gate = (margin > 0.0).astype(np.float64) if hard else expit(margin)
        bend = (sigmoid_prime(margin) * (ddelta * (delta < 0.0)))[:, None]
        return gate[:, None] * dx + (1.0 - gate)[:, None] * V + (x - S) * bend

    def _jvp_batch(self, ts, S, V):
        return self._tangent(ts, S, V, True)

    def relaxed_jvp_batch(self, ts, S, V):
        return self._tangent(np.asarray(ts), np.asarray(S, dtype=np.float64),
                             np.asarray(V, dtype=np.float64), False)


# ---------------------------------------------------------------------------
# eight schools Gibbs (samplers.py:416-668)

HYPER = dict(nu0=0.1, tau0_sq=100.0, mu0=0.0, kappa0=0.1, alpha0=0.1, sigma0_sq=10.0)
EFFECTS = (28.0, 8.0, -3.0, 7.0, -1.0, 1.0, 18.0, 12.0)
SES = (15.0, 10.0, 16.0, 11.0, 9.0, 11.0, 10.0, 18.0)


class SchoolsData:
    def __init__(self, x):
        self.x = np.asarray(x, dtype=np.float64)
        self.n_schools, self.n_per_school = self.x.shape
        self.xbar = self.x.mean(axis=1)
        self.ss = np.sum((self.x - self.xbar[:, None]) ** 2, axis=1)


def generate_eight_schools(seed=11, n_per_school=20):
    """Per-school rows rescaled to the classic means/SEs (samplers.py:445-461)."""
    tab = NoiseTable(seed, {"z": SlotSpec(n_per_school, "standard-normal")}, T=len(EFFECTS))
    rows = []
    for s, (eff, se) in enumerate(zip(EFFECTS, SES)):
        z = tab.block("z", np.array([s + 1]))[0]
        z = z - z.mean()
        z = z / z.std(ddof=1)
        rows.append(eff + z * se * np.sqrt(n_per_school))
    return SchoolsData(np.array(rows))


class GibbsKernel(System):
    """Systematic sweep tau^2, mu, theta, sigma^2 on fixed noise."""

    FLOOR = 1e-8

    def __init__(self, data, hyper=None, seed=0, T=1):
        h = dict(HYPER if hyper is None else hyper)
        S = data.n_schools
        layout = {
            "g_tau": SlotSpec(1, "chi-squared", df=h["nu0"] + S + 1),
            "xi_mu": SlotSpec(1, "standard-normal"),
            "xi_theta": SlotSpec(S, "standard-normal"),
            "g_sigma": SlotSpec(S, "chi-squared", df=h["alpha0"] + data.n_per_school),
            "g_tau_prior": SlotSpec(1, "chi-squared", df=h["nu0"]),
            "xi_mu_prior": SlotSpec(1, "standard-normal"),
            "xi_theta_prior": SlotSpec(S, "standard-normal"),
            "g_sigma_prior": SlotSpec(S, "chi-squared", df=h["alpha0"]),
        }
        super().__init__(2 * S + 2, NoiseTable(seed, layout, T))
        self.data, self.h, self.S = data, h, S
        self._cache = {}

    def recommended_preconditioner(self):
        pre = np.ones(self.dim)
        pre[0] = 1e-12
        pre[2 + self.S:] = 1e-12
        return pre

    def _noise(self, ts):
        key = np.asarray(ts).tobytes()
        if key not in self._cache:
            if len(self._cache) >= 4:
                self._cache.pop(next(iter(self._cache)))
            self._cache[key] = {k: self.noise.block(k, ts)
                                for k in ("g_tau", "xi_mu", "xi_theta", "g_sigma")}
        return self._cache[key]

    def _split(self, st):
        S = self.S
        return st[..., 0], st[..., 1], st[..., 2:2 + S], st[..., 2 + S:]

    def sweep(self, ts, state):
        h, d, S = self.h, self.data, self.S
        _, mu, th, sg = self._split(np.asarray(state, dtype=np.float64))
        sg = np.maximum(sg, self.FLOOR)
        nz = self._noise(ts)
        g_tau, xi_mu, xi_th, g_sig = nz["g_tau"][:, 0], nz["xi_mu"][:, 0], nz["xi_theta"], nz["g_sigma"]
        q_tau = h["nu0"] * h["tau0_sq"] + h["kappa0"] * (mu - h["mu0"]) ** 2 \
            + np.sum((th - mu[:, None]) ** 2, axis=-1)
        tau2 = q_tau / g_tau
        kS = h["kappa0"] + S
        mu_n = (h["kappa0"] * h["mu0"] + th.sum(axis=-1)) / kS + np.sqrt(tau2 / kS) * xi_mu
        n = d.n_per_school
        prec = 1.0 / tau2[:, None] + n / sg
        mean = (mu_n[:, None] / tau2[:, None] + n * d.xbar / sg) / prec
        th_n = mean + xi_th / np.sqrt(prec)
        sg_n = (h["alpha0"] * h["sigma0_sq"] + d.ss + n * (d.xbar - th_n) ** 2) / g_sig
        return dict(mu=mu, th=th, sg=sg, g_tau=g_tau, xi_mu=xi_mu, xi_th=xi_th, g_sig=g_sig,
                    tau2=tau2, mu_n=mu_n, prec=prec, mean=mean, th_n=th_n, sg_n=sg_n)

    def _step_batch(self, ts, state):
        f = self.sweep(ts, state)
        return np.concatenate([f["tau2"][:, None], f["mu_n"][:, None], f["th_n"], f["sg_n"]], axis=-1)

    def _jvp_batch(self, ts, state, V):
        h, d, S = self.h, self.data, self.S
        n = d.n_per_school
        f = self.sweep(ts, state)
        _, dmu_in, dth_in, dsg_in = self._split(V)
        raw_sg = self._split(np.asarray(state, dtype=np.float64))[3]
        dsg_in = np.where(raw_sg > self.FLOOR, dsg_in, 0.0)
        dq = 2.0 * h["kappa0"] * (f["mu"] - h["mu0"]) * dmu_in + np.sum(
            2.0 * (f["th"] - f["mu"][:, None]) * (dth_in - dmu_in[:, None]), axis=-1)
        dtau2 = dq / f["g_tau"]
        kS = h["kappa0"] + S
        dmu = dth_in.sum(axis=-1) / kS + f["xi_mu"] * dtau2 / (2.0 * np.sqrt(f["tau2"] * kS))
        t2 = f["tau2"][:, None]
        dt2 = dtau2[:, None]
        dprec = -dt2 / t2 ** 2 - n * dsg_in / f["sg"] ** 2
        damean = dmu[:, None] / t2 - f["mu_n"][:, None] * dt2 / t2 ** 2 - n * d.xbar * dsg_in / f["sg"] ** 2
        dmean = (damean - f["mean"] * dprec) / f["prec"]
        dth = dmean - 0.5 * f["xi_th"] * dprec / f["prec"] ** 1.5
        dsg = (-2.0 * n * (d.xbar - f["th_n"]) * dth) / f["g_sig"]
        return np.concatenate([dtau2[:, None], dmu[:, None], dth, dsg], axis=-1)

    def initial_state(self):
        """Prior draw at t=0 then one sweep step(0, .) (samplers.py:631-641)."""
        h = self.h
        t0 = np.array([0])
        tau2 = h["nu0"] * h["tau0_sq"] / self.noise.block("g_tau_prior", t0)[0, 0]
        mu = h["mu0"] + np.sqrt(tau2 / h["kappa0"]) * self.noise.block("xi_mu_prior", t0)[0, 0]
        th = mu + np.sqrt(tau2) * self.noise.block("xi_theta_prior", t0)[0]
        sg = h["alpha0"] * h["sigma0_sq"] / self.noise.block("g_sigma_prior", t0)[0]
        prior = np.concatenate([[tau2], [mu], th, sg])
        return self.step(0, prior)

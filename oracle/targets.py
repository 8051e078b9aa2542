"""Target log-densities with analytic grad / Hessian-vector products
(TEST INFRASTRUCTURE ONLY).

Reference: ``chainscan/targets.py`` -- std-normal (160-166), Gaussian given the
Cholesky factor of its precision (169-182), Rosenbrock banana (185-212),
isotropic mixture of Gaussians (215-251), Bayesian logistic regression with a
spherical prior, evaluated in row tiles of 4M logits (254-287); the synthetic
credit-like dataset (376-396).  All methods broadcast over leading axes.
"""

from __future__ import annotations

import numpy as np
from scipy.special import expit

from .errors import ConfigurationError, StructuralError
from .rng import NoiseTable, SlotSpec

BLR_TILE_ELEMENTS = 4_000_000


class Target:
    """kind in {std-normal, gaussian, rosenbrock, mog, blr}; params per kind."""

    def __init__(self, kind, dim, **params):
        self.kind = kind
        self.dim = int(dim)
        self.params = params
        if kind == "gaussian":
            L = params["chol_precision"]
            self.P = L @ L.T
        if kind == "mog":
            self.logw = np.log(params["weights"])
            self.lognorm = -0.5 * self.dim * np.log(2 * np.pi * params["variances"])

    # -- per family ---------------------------------------------------------
    def logp(self, x):
        x = np.asarray(x, dtype=np.float64)
        k, p = self.kind, self.params
        if k == "std-normal":
            return -0.5 * np.sum(x * x, axis=-1)
        if k == "gaussian":
            h = (x - p["mu"]) @ p["chol_precision"]
            return -0.5 * np.sum(h * h, axis=-1)
        if k == "rosenbrock":
            x1, x2 = x[..., 0], x[..., 1]
            r = x2 - p["b"] * x1 * x1
            return -((x1 - p["a"]) ** 2) / (2 * p["scale1"]) - r * r / (2 * p["scale2"])
        if k == "mog":
            lc, _ = self._components(x)
            top = lc.max(axis=-1)
            return top + np.log(np.sum(np.exp(lc - top[..., None]), axis=-1))
        return self._blr_tiles(x, "logp")

    def grad(self, x):
        x = np.asarray(x, dtype=np.float64)
        k, p = self.kind, self.params
        if k == "std-normal":
            return -x
        if k == "gaussian":
            return -((x - p["mu"]) @ self.P)
        if k == "rosenbrock":
            x1, x2 = x[..., 0], x[..., 1]
            b, s1, s2 = p["b"], p["scale1"], p["scale2"]
            r = x2 - b * x1 * x1
            return np.stack([-(x1 - p["a"]) / s1 + 2 * b * x1 * r / s2, -r / s2], axis=-1)
        if k == "mog":
            resp, diff = self._resp(x)
            return -np.sum(resp[..., None] * diff / p["variances"][:, None], axis=-2)
        return self._blr_tiles(x, "grad")

    def hvp(self, x, v):
        x = np.asarray(x, dtype=np.float64)
        v = np.asarray(v, dtype=np.float64)
        k, p = self.kind, self.params
        if k == "std-normal":
            return -v
        if k == "gaussian":
            return -(v @ self.P)
        if k == "rosenbrock":
            x1, x2 = x[..., 0], x[..., 1]
            b, s1, s2 = p["b"], p["scale1"], p["scale2"]
            r = x2 - b * x1 * x1
            h11 = -1.0 / s1 + (2 * b * r - 4 * b * b * x1 * x1) / s2
            h12 = 2 * b * x1 / s2
            return np.stack([h11 * v[..., 0] + h12 * v[..., 1],
                             h12 * v[..., 0] - v[..., 1] / s2], axis=-1)
        if k == "mog":
            var = p["variances"]
            resp, diff = self._resp(x)
            gk = -diff / var[:, None]
            gbar = np.sum(resp[..., None] * gk, axis=-2)
            gv = np.sum(gk * v[..., None, :], axis=-1)
            term = np.sum((resp * gv)[..., None] * gk, axis=-2)
            curv = np.sum(resp / var, axis=-1)
            return term - curv[..., None] * v - gbar * np.sum(gbar * v, axis=-1)[..., None]
        return self._blr_tiles(x, "hvp", v)

    # -- helpers --------------------------------------------------------------
    def _components(self, x):
        diff = x[..., None, :] - self.params["means"]
        sq = np.sum(diff * diff, axis=-1)
        return self.logw + self.lognorm - sq / (2 * self.params["variances"]), diff

    def _resp(self, x):
        lc, diff = self._components(x)
        e = np.exp(lc - lc.max(axis=-1, keepdims=True))
        return e / e.sum(axis=-1, keepdims=True), diff

    def _blr_tiles(self, beta, what, v=None):
        X, y, prec = self.params["X"], self.params["y"], self.params["prior_precision"]
        n, d = X.shape
        if beta.shape[-1] != d:
            raise StructuralError("trailing dimension mismatch")
        lead = beta.shape[:-1]
        flat = beta.reshape(-1, d)
        rows = max(1, BLR_TILE_ELEMENTS // max(n, 1))
        if what == "logp":
            out = np.empty(flat.shape[0])
            for lo in range(0, flat.shape[0], rows):
                eta = flat[lo:lo + rows] @ X.T
                out[lo:lo + rows] = eta @ y - np.logaddexp(0.0, eta).sum(axis=-1)
            out -= 0.5 * prec * np.sum(flat * flat, axis=-1)
            return out.reshape(lead)
        out = np.empty_like(flat)
        if what == "grad":
            for lo in range(0, flat.shape[0], rows):
                out[lo:lo + rows] = (y - expit(flat[lo:lo + rows] @ X.T)) @ X
            out -= prec * flat
            return out.reshape(lead + (d,))
        vflat = np.broadcast_to(v, beta.shape).reshape(-1, d)
        for lo in range(0, flat.shape[0], rows):
            pr = expit(flat[lo:lo + rows] @ X.T)
            xv = vflat[lo:lo + rows] @ X.T
            out[lo:lo + rows] = -((pr * (1.0 - pr) * xv) @ X)
        out -= prec * vflat
        return out.reshape(lead + (d,))


def std_normal(dim):
    return Target("std-normal", dim)


def gaussian(mu, chol_precision):
    mu = np.asarray(mu, dtype=np.float64)
    L = np.asarray(chol_precision, dtype=np.float64)
    if mu.ndim != 1 or L.shape != (mu.size, mu.size) or np.any(np.diag(L) <= 0):
        raise ConfigurationError("bad gaussian parameters")
    return Target("gaussian", mu.size, mu=mu, chol_precision=L)


def rosenbrock(a=0.0, b=1.0, scale1=1.0, scale2=0.1):
    if scale1 <= 0 or scale2 <= 0:
        raise ConfigurationError("rosenbrock scales must be positive")
    return Target("rosenbrock", 2, a=float(a), b=float(b), scale1=float(scale1),
                  scale2=float(scale2))


def mog(weights=None, means=None, variances=None):
    if means is None:
        means = [(-3.0, -3.0), (-3.0, 3.0), (3.0, -3.0), (3.0, 3.0)]
    means = np.asarray(means, dtype=np.float64)
    K = means.shape[0]
    weights = np.full(K, 1.0 / K) if weights is None else np.asarray(weights, dtype=np.float64)
    variances = np.ones(K) if variances is None else np.asarray(variances, dtype=np.float64)
    return Target("mog", means.shape[1], weights=weights, means=means, variances=variances)


def blr(X, y, prior_precision=1.0):
    X = np.asarray(X, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    if X.ndim != 2 or y.shape != (X.shape[0],) or prior_precision <= 0:
        raise ConfigurationError("bad logistic-regression data")
    return Target("blr", X.shape[1], X=X, y=y, prior_precision=float(prior_precision))


def synthetic_credit_like(seed=20250819, n=1000, dim=25):
    """N(0,1) features, beta* from t=0, y ~ Bernoulli(sigmoid(X beta*)) (targets.py:376-396)."""
    tab = NoiseTable(seed, {"x": SlotSpec(dim, "standard-normal"),
                            "u": SlotSpec(1, "uniform-0-1"),
                            "beta": SlotSpec(dim, "standard-normal")}, T=n)
    beta_star = tab.block("beta", [0])[0]
    rows = np.arange(1, n + 1)
    X = tab.block("x", rows)
    u = tab.block("u", rows)[:, 0]
    y = (u < expit(X @ beta_star)).astype(np.float64)
    return X, y, beta_star

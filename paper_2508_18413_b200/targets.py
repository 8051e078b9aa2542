"""Target log-densities (mirror of chainscan/targets.py).

A ``ModelSpec`` (targets.py:57-71) is validated exactly like the reference's.
``model_logp_grad_hvp`` compiles it into a ``TargetModel`` whose parameters
live in HBM and which carries the ``cs_target`` descriptor the fused CUDA
sampler kernels read; the batched ``logp/grad/hvp`` callables are device
tensor programs for API parity and tests (the fused kernels never call them).
Logistic regression evaluates its data contractions as cuBLAS GEMMs.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field
from typing import Any

import numpy as np
import torch

from . import _lib
from .core import StructuralError, TargetModel
from .errors import ConfigurationError
from .noise import NoiseTable, SlotSpec

__all__ = ["ModelSpec", "std_normal", "gaussian", "rosenbrock", "mog", "blr",
           "model_logp_grad_hvp", "synthetic_credit_like", "MODEL_KINDS"]

MODEL_KINDS = ("std-normal", "gaussian", "rosenbrock", "mog", "blr")
_KIND_CODE = {"std-normal": _lib.CS_TARGET_STD_NORMAL, "gaussian": _lib.CS_TARGET_GAUSSIAN,
              "rosenbrock": _lib.CS_TARGET_ROSENBROCK, "mog": _lib.CS_TARGET_MOG,
              "blr": _lib.CS_TARGET_BLR}


@dataclass(frozen=True)
class ModelSpec:
    kind: str
    dim: int
    params: dict[str, Any] = field(default_factory=dict)

    def __post_init__(self):
        if self.kind not in MODEL_KINDS:
            raise ConfigurationError(f"unknown model kind {self.kind!r}; expected one of {MODEL_KINDS}")
        if self.dim < 1:
            raise ConfigurationError(f"model dim must be >= 1, got {self.dim}")


def std_normal(dim: int) -> ModelSpec:
    return ModelSpec("std-normal", int(dim))


def gaussian(mu, chol_precision) -> ModelSpec:
    """Gaussian with mean mu and precision L L^T given by its factor L (targets.py:78-89)."""
    mu = np.asarray(mu, float)
    L = np.asarray(chol_precision, float)
    if mu.ndim != 1:
        raise ConfigurationError(f"mu must be a vector, got shape {mu.shape}")
    d = mu.shape[0]
    if L.shape != (d, d):
        raise ConfigurationError(f"chol_precision must be {d}x{d}, got {L.shape}")
    if not np.all(np.isfinite(L)) or np.any(np.diag(L) <= 0):
        raise ConfigurationError("chol_precision needs a positive diagonal")
    return ModelSpec("gaussian", d, {"mu": mu, "chol_precision": L})


def rosenbrock(a=0.0, b=1.0, scale1=1.0, scale2=0.1) -> ModelSpec:
    if scale1 <= 0 or scale2 <= 0:
        raise ConfigurationError("rosenbrock scales must be positive")
    return ModelSpec("rosenbrock", 2, {"a": float(a), "b": float(b), "scale1": float(scale1),
                                       "scale2": float(scale2)})


def mog(weights=None, means=None, variances=None) -> ModelSpec:
    if means is None:
        means = [(-3.0, -3.0), (-3.0, 3.0), (3.0, -3.0), (3.0, 3.0)]
    means = np.asarray(means, float)
    if means.ndim != 2:
        raise ConfigurationError(f"means must be (K, D), got shape {means.shape}")
    K, d = means.shape
    weights = np.full(K, 1.0 / K) if weights is None else np.asarray(weights, float)
    variances = np.ones(K) if variances is None else np.asarray(variances, float)
    if weights.shape != (K,) or variances.shape != (K,):
        raise ConfigurationError("weights/variances must have one entry per component")
    if np.any(weights <= 0) or abs(weights.sum() - 1.0) > 1e-9:
        raise ConfigurationError("weights must be positive and sum to 1")
    if np.any(variances <= 0):
        raise ConfigurationError("variances must be positive")
    return ModelSpec("mog", d, {"weights": weights, "means": means, "variances": variances})


def blr(X, y, prior_precision=1.0) -> ModelSpec:
    X = np.asarray(X, float)
    y = np.asarray(y, float)
    if X.ndim != 2:
        raise ConfigurationError(f"X must be (N, D), got shape {X.shape}")
    if y.shape != (X.shape[0],):
        raise ConfigurationError(f"labels must match rows: X has {X.shape[0]}, y has shape {y.shape}")
    if not np.all(np.isin(y, (0.0, 1.0))):
        raise ConfigurationError("labels must be 0/1")
    if prior_precision <= 0:
        raise ConfigurationError("prior precision must be positive")
    return ModelSpec("blr", X.shape[1], {"X": X, "y": y, "prior_precision": float(prior_precision)})


class DeviceTarget(TargetModel):
    pass


def _dev():
    _lib.require_cuda()
    return torch.device("cuda", torch.cuda.current_device())


def _t(x, dev):
    return torch.as_tensor(np.ascontiguousarray(x, dtype=np.float64), device=dev)


def _flat(x, dim):
    if x.shape[-1] != dim:
        raise StructuralError(f"expected trailing dimension {dim}, got shape {tuple(x.shape)}")
    return x.reshape(-1, dim), x.shape[:-1]


def _native(desc, what, dim, x, v=None):
    """log density (what 0), gradient (1) or Hessian-vector product (2) of a
    GEMM-shaped target for a batch of states, through cs_target_eval."""
    flat, lead = _flat(x, dim)
    flat = flat.contiguous()
    n = flat.shape[0]
    vflat = None
    if v is not None:
        vflat = _flat(v.expand(x.shape), dim)[0].contiguous()
    out = torch.empty((n,) if what == 0 else (n, dim), dtype=torch.float64, device=flat.device)
    _lib.check(_lib.load().cs_target_eval(ctypes.byref(desc), what, n, _lib.ptr(flat), _lib.ptr(vflat),
                                          _lib.ptr(out), _lib.stream_ptr()))
    return out.reshape(lead) if what == 0 else out.reshape(tuple(lead) + (dim,))


def model_logp_grad_hvp(spec: ModelSpec) -> TargetModel:
    """Compile a ModelSpec (targets.py:290-308): device parameters + cs_target."""
    dev = _dev()
    p = spec.params
    keep = {}
    desc = _lib.cs_target()
    desc.kind = _KIND_CODE[spec.kind]
    desc.dim = spec.dim

    def f64(x):
        return torch.as_tensor(x, dtype=torch.float64, device=dev)

    if spec.kind == "std-normal":
        logp = lambda x: -0.5 * torch.sum(f64(x) ** 2, dim=-1)
        grad = lambda x: -f64(x)
        hvp = lambda x, v: -f64(v)
    elif spec.kind == "gaussian":
        mu_np, L_np = p["mu"], p["chol_precision"]
        P_np = L_np @ L_np.T          # same BLAS product as targets.py:170
        mu, L, P = _t(mu_np, dev), _t(L_np, dev), _t(P_np, dev)
        keep.update(mu=mu, L=L, P=P)
        desc.mu, desc.chol, desc.prec = mu.data_ptr(), L.data_ptr(), P.data_ptr()

        # the library's DMMA GEMM (cs_target_eval): same arithmetic as
        # targets.py:168-180, no vendor BLAS
        logp = lambda x: _native(desc, 0, spec.dim, f64(x))
        grad = lambda x: _native(desc, 1, spec.dim, f64(x))
        hvp = lambda x, v: _native(desc, 2, spec.dim, f64(x), f64(v))
    elif spec.kind == "rosenbrock":
        a, b, s1, s2 = p["a"], p["b"], p["scale1"], p["scale2"]
        desc.a, desc.b, desc.scale1, desc.scale2 = a, b, s1, s2

        def logp(x):
            x = f64(x)
            x1, x2 = x[..., 0], x[..., 1]
            r = x2 - b * x1 * x1
            return -((x1 - a) ** 2) / (2 * s1) - r * r / (2 * s2)

        def grad(x):
            x = f64(x)
            x1, x2 = x[..., 0], x[..., 1]
            r = x2 - b * x1 * x1
            return torch.stack([-(x1 - a) / s1 + 2 * b * x1 * r / s2, -r / s2], dim=-1)

        def hvp(x, v):
            x, v = f64(x), f64(v)
            x1, x2 = x[..., 0], x[..., 1]
            r = x2 - b * x1 * x1
            h11 = -1.0 / s1 + (2 * b * r - 4 * b * b * x1 * x1) / s2
            h12 = 2 * b * x1 / s2
            return torch.stack([h11 * v[..., 0] + h12 * v[..., 1], h12 * v[..., 0] - v[..., 1] / s2], dim=-1)
    elif spec.kind == "mog":
        w, m_np, var_np = p["weights"], p["means"], p["variances"]
        d = m_np.shape[1]
        logw_np = np.log(w)
        lognorm_np = -0.5 * d * np.log(2 * np.pi * var_np)
        means, var, logw, lognorm = _t(m_np, dev), _t(var_np, dev), _t(logw_np, dev), _t(lognorm_np, dev)
        keep.update(means=means, var=var, logw=logw, lognorm=lognorm)
        desc.n_comp = m_np.shape[0]
        desc.means, desc.variances = means.data_ptr(), var.data_ptr()
        desc.logw, desc.lognorm = logw.data_ptr(), lognorm.data_ptr()

        def comps(x):
            diff = x[..., None, :] - means
            sq = torch.sum(diff * diff, dim=-1)
            return logw + lognorm - sq / (2 * var), diff

        def logp(x):
            lc, _ = comps(f64(x))
            mx = lc.max(dim=-1).values
            return mx + torch.log(torch.sum(torch.exp(lc - mx[..., None]), dim=-1))

        def resp(x):
            lc, diff = comps(x)
            e = torch.exp(lc - lc.max(dim=-1, keepdim=True).values)
            return e / e.sum(dim=-1, keepdim=True), diff

        def grad(x):
            r, diff = resp(f64(x))
            return -torch.sum(r[..., None] * diff / var[:, None], dim=-2)

        def hvp(x, v):
            x, v = f64(x), f64(v)
            r, diff = resp(x)
            gk = -diff / var[:, None]
            gbar = torch.sum(r[..., None] * gk, dim=-2)
            gv = torch.sum(gk * v[..., None, :], dim=-1)
            term = torch.sum((r * gv)[..., None] * gk, dim=-2)
            curv = torch.sum(r / var, dim=-1)
            return term - curv[..., None] * v - gbar * torch.sum(gbar * v, dim=-1)[..., None]
    else:  # blr (targets.py:254-287): eta = beta X^T and the products against X on the library's DMMA GEMM
        X, y, prec = _t(p["X"], dev), _t(p["y"], dev), p["prior_precision"]
        keep.update(X=X, y=y)
        desc.n_data = X.shape[0]
        desc.X, desc.y, desc.prior_precision = X.data_ptr(), y.data_ptr(), prec
        logp = lambda beta: _native(desc, 0, spec.dim, f64(beta))
        grad = lambda beta: _native(desc, 1, spec.dim, f64(beta))
        hvp = lambda beta, v: _native(desc, 2, spec.dim, f64(beta), f64(v))

    tm = DeviceTarget(dim=spec.dim, logp=logp, grad=grad, hvp=hvp, spec=spec)
    object.__setattr__(tm, "_keep", keep)
    object.__setattr__(tm, "desc", desc)
    return tm


def synthetic_credit_like(seed: int = 20250819, n: int = 1000, dim: int = 25):
    """Deterministic logistic-regression data (targets.py:376-396), drawn on device.

    Returns numpy (X, y, beta_star) like the reference.
    """
    table = NoiseTable(seed, {"x": SlotSpec(dim, "standard-normal"), "u": SlotSpec(1, "uniform-0-1"),
                              "beta": SlotSpec(dim, "standard-normal")}, T=n)
    beta = table.fill("beta", 0, 1)[0]
    X = table.fill("x", 1, n)
    u = table.fill("u", 1, n)[:, 0]
    y = (u < torch.sigmoid(X @ beta)).to(torch.float64)
    return X.cpu().numpy(), y.cpu().numpy(), beta.cpu().numpy()

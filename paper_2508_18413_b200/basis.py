"""Orthogonal change of basis for a transition system (targets.py:400-517).

``orthogonal_basis(C)`` eigendecomposes a symmetric matrix on the device
(cuSOLVER through torch.linalg.eigh; the reference uses cyclic Jacobi
rotations) and returns the same canonical form: eigenvalues descending, each
column sign-fixed so its largest-magnitude entry is positive.  For distinct
eigenvalues that pins the basis uniquely, so results agree with the
reference's to rounding.  ``transform_system(system, Q)`` conjugates a system
into z = Q' s coordinates, z -> Q' f(Q z), with jvp and dense Jacobian
conjugated alike; solving it from Q' s0 and mapping back through Q reproduces
the original trace (quasi-Newton solves converge faster on correlated targets
in the eigenbasis).  For the built-in MALA / HMC systems Q
is fused into the CUDA kernels (the system descriptor carries it; f_t,
tangents, the sequential walk and the streamed engine's element builder
conjugate in registers); other systems get the conjugation as batched GEMMs
around their step / jvp calls.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .core import TransitionSystem, as_steps
from .errors import StructuralError

__all__ = ["OrthogonalBasis", "orthogonal_basis", "transform_system"]


@dataclass(frozen=True)
class OrthogonalBasis:
    """Columns of Q are orthonormal; eigenvalues sorted descending (targets.py:403-414)."""

    Q: torch.Tensor
    eigenvalues: torch.Tensor

    def __post_init__(self):
        d = self.Q.shape[0]
        err = float((self.Q.T @ self.Q - torch.eye(d, dtype=self.Q.dtype, device=self.Q.device)).abs().max()) \
            if d else 0.0
        if err > 1e-10:
            raise StructuralError(f"basis is not orthogonal: max |Q'Q - I| = {err:.2e}")


def _device(device):
    return torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())


def orthogonal_basis(C, device=None) -> OrthogonalBasis:
    """Eigenbasis of a symmetric matrix in the reference's canonical form (targets.py:417-467)."""
    C = torch.as_tensor(np.asarray(C, float) if not torch.is_tensor(C) else C, dtype=torch.float64,
                        device=_device(device) if not torch.is_tensor(C) else C.device)
    if C.ndim != 2 or C.shape[0] != C.shape[1]:
        raise StructuralError(f"expected a square matrix, got shape {tuple(C.shape)}")
    scale = max(1.0, float(C.abs().max())) if C.numel() else 1.0
    if C.numel() and float((C - C.T).abs().max()) > 1e-10 * scale:
        raise StructuralError("matrix is not symmetric")
    evals, Q = torch.linalg.eigh(0.5 * (C + C.T))
    order = torch.argsort(-evals, stable=True)
    evals, Q = evals[order], Q[:, order].contiguous()
    if Q.numel():
        big = Q.abs().argmax(dim=0)
        sign = torch.where(Q[big, torch.arange(Q.shape[1], device=Q.device)] < 0, -1.0, 1.0).to(Q.dtype)
        Q = Q * sign[None, :]
    return OrthogonalBasis(Q=Q, eigenvalues=evals)


class _TransformedSystem(TransitionSystem):
    """The base system conjugated into z = Q' s coordinates (targets.py:470-501)."""

    def __init__(self, base: TransitionSystem, Q: torch.Tensor):
        super().__init__(base.dim, base.noise, dtype=base.dtype, device=base.device)
        self.base = base
        self.Q = Q.to(dtype=base.dtype, device=base.device)

    def transform_state(self, s):
        return torch.as_tensor(s, dtype=self.dtype, device=self.device) @ self.Q

    def untransform_state(self, z):
        return torch.as_tensor(z, dtype=self.dtype, device=self.device) @ self.Q.T

    def _step_batch(self, ts, Z):
        return self.base.step_batch(ts, Z @ self.Q.T) @ self.Q

    def _jvp_batch(self, ts, Z, V):
        return self.base.jvp_batch(ts, Z @ self.Q.T, V @ self.Q.T) @ self.Q

    def relaxed_step_batch(self, ts, Z):
        return self.base.relaxed_step_batch(ts, self._state(Z) @ self.Q.T) @ self.Q

    def relaxed_jvp_batch(self, ts, Z, V):
        return self.base.relaxed_jvp_batch(ts, self._state(Z) @ self.Q.T, self._state(V) @ self.Q.T) @ self.Q

    def dense_jacobian_batch(self, ts, Z):
        J = self.base.dense_jacobian_batch(as_steps(ts, self.device), self._state(Z) @ self.Q.T)
        return self.Q.T @ J @ self.Q


class _FusedTransformed(_TransformedSystem):
    """A built-in MALA / HMC system in z = Q' s coordinates with Q fused into its
    CUDA kernels: the descriptor carries Q, so f_t, the tangents, the sequential
    walk and the streamed engine's element builder conjugate in registers
    (x = Q z on the way in, Q' on the way out) -- no extra passes over T."""

    def __init__(self, base, Q):
        super().__init__(base, Q)
        from .samplers import _Fused

        self._Qd = Q.to(dtype=torch.float64, device=base.device).contiguous()
        self._kind = base._kind
        self._what = base._what
        self._call_step = _Fused._call_step.__get__(self)
        self._call_jvp = _Fused._call_jvp.__get__(self)
        self._sequential_kernel = _Fused._sequential_kernel.__get__(self)

    def desc(self):
        d = self.base.desc()
        d.basis = self._Qd.data_ptr()
        return d

    @property
    def kernels(self) -> bool:
        return True

    @property
    def _sequential(self):
        return self._sequential_kernel

    def _step_batch(self, ts, Z):
        return self._call_step(ts, Z)

    def _jvp_batch(self, ts, Z, V):
        return self._call_jvp(ts, Z, V)

    def relaxed_step_batch(self, ts, Z):
        return self._call_step(as_steps(ts, self.device), self._state(Z), relaxed=True)

    def relaxed_jvp_batch(self, ts, Z, V):
        return self._call_jvp(as_steps(ts, self.device), self._state(Z), self._state(V), relaxed=True)

    def dense_jacobian_batch(self, ts, Z):
        return TransitionSystem.dense_jacobian_batch(self, ts, Z)


def _fusable(system) -> bool:
    from . import _lib
    from .samplers import HmcKernel, MalaKernel

    if not isinstance(system, (MalaKernel, HmcKernel)) or not getattr(system, "kernels", False):
        return False
    if getattr(system, "leapfrog_mode", "sequential") == "parallel":
        return False
    import ctypes

    d = system.desc()
    probe = torch.eye(system.dim, dtype=torch.float64, device=system.device)
    d.basis = probe.data_ptr()
    return bool(_lib.load().cs_system_supported(ctypes.byref(d), _lib.dtype_code(system.dtype)))


def transform_system(system: TransitionSystem, Q) -> TransitionSystem:
    """Rewrite a system in the orthogonal coordinates z = Q' s (targets.py:504-517)."""
    Q = torch.as_tensor(np.asarray(Q, float) if not torch.is_tensor(Q) else Q, dtype=torch.float64,
                        device=system.device)
    d = system.dim
    if tuple(Q.shape) != (d, d):
        raise StructuralError(f"Q must be {d}x{d} to match the system, got {tuple(Q.shape)}")
    if float((Q.T @ Q - torch.eye(d, dtype=Q.dtype, device=Q.device)).abs().max()) > 1e-10:
        raise StructuralError("Q is not orthogonal")
    if _fusable(system):
        return _FusedTransformed(system, Q)
    return _TransformedSystem(system, Q)

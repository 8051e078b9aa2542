"""Affine scan elements and the parallel solver for linear recursions
(mirror of chainscan/pscan.py) on B200.

An element (J_t, u_t) maps s -> J_t s + u_t in one of three carriers:
Diag (j, u), Dense (J, u), Block2x2 (a, b, c, d, u) on a stacked [x, v] state
(pscan.py:100-173).  ``parallel_affine_solve`` runs the CUDA scans of
csrc/cs_scan.cu: chunks of rows reduced and replayed with f64 carries, linked
by look-back.  Every chunk's entry state is the fixed chain
exit(k) = A_k(exit(k-1)) from s0 -- the look-back applies the aggregates it
needs one at a time instead of composing them first -- so for a given shape
the result is bit-identical run to run however the look-back races resolve
(the reference's fixed-chunk property, _scan_kernels.py:3-8;
tests/test_parity_baseline_gpu.py::test_scan_bit_identical_run_to_run).
``workers`` / ``chunk`` are accepted for API compatibility; the device tiling
depends only on the shape.
"""

from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass

import torch

from . import _lib
from .core import StructuralError

__all__ = ["DiagElements", "DenseElements", "Block2x2Elements", "identity_element", "compose",
           "apply_element", "sequential_affine_solve", "parallel_affine_solve", "set_workers",
           "get_workers", "max_hardware_workers", "default_chunk"]


def _env_workers() -> int:
    raw = os.environ.get("CHAINSCAN_THREADS", "")
    if raw:
        try:
            n = int(raw)
            if n >= 1:
                return n
        except ValueError:
            pass
    return os.cpu_count() or 1


_WORKERS = _env_workers()


def max_hardware_workers() -> int:
    return os.cpu_count() or 1


def set_workers(n: int) -> int:
    """Kept for API compatibility (pscan.py:69-84); drives default_chunk only."""
    global _WORKERS
    n = int(n)
    if n < 1:
        raise ValueError(f"workers must be >= 1, got {n}")
    _WORKERS = n
    return _WORKERS


def get_workers() -> int:
    return _WORKERS


def default_chunk(T: int, workers: int) -> int:
    """The reference's CPU chunk policy (pscan.py:269-270)."""
    return max(min(T, 256), math.ceil(T / (8 * workers)))


def _tensor(x, like=None):
    if torch.is_tensor(x):
        return x
    dev = like.device if like is not None else torch.device("cuda", torch.cuda.current_device())
    dt = like.dtype if like is not None else torch.float64
    return torch.as_tensor(x, dtype=dt, device=dev)


def _unify(*ts):
    """Common floating dtype (f64 wins, like the reference's np.asarray(float))."""
    dt = torch.float64 if any(t.dtype == torch.float64 for t in ts) else torch.float32
    dev = ts[0].device
    return [t.to(device=dev, dtype=dt) for t in ts]


def _same(a, b, what):
    if tuple(a.shape) != tuple(b.shape):
        raise StructuralError(f"{what}: shapes {tuple(a.shape)} and {tuple(b.shape)} differ")


@dataclass
class DiagElements:
    j: torch.Tensor
    u: torch.Tensor

    def __post_init__(self):
        self.j, self.u = _unify(_tensor(self.j), _tensor(self.u))
        _same(self.j, self.u, "Diag j/u")

    @property
    def dim(self) -> int:
        return self.j.shape[-1]

    def nbytes(self) -> int:
        return self.j.numel() * self.j.element_size() + self.u.numel() * self.u.element_size()


@dataclass
class DenseElements:
    J: torch.Tensor
    u: torch.Tensor

    def __post_init__(self):
        self.J, self.u = _unify(_tensor(self.J), _tensor(self.u))
        if self.J.shape[-1] != self.J.shape[-2]:
            raise StructuralError(f"Dense J must be square, got {tuple(self.J.shape)}")
        _same(self.J[..., 0], self.u, "Dense J/u")

    @property
    def dim(self) -> int:
        return self.J.shape[-1]

    def nbytes(self) -> int:
        return self.J.numel() * self.J.element_size() + self.u.numel() * self.u.element_size()


@dataclass
class Block2x2Elements:
    a: torch.Tensor
    b: torch.Tensor
    c: torch.Tensor
    d: torch.Tensor
    u: torch.Tensor

    def __post_init__(self):
        self.a, self.b, self.c, self.d, self.u = _unify(
            *(_tensor(getattr(self, n)) for n in ("a", "b", "c", "d", "u")))
        for name in ("b", "c", "d"):
            _same(self.a, getattr(self, name), f"Block2x2 a/{name}")
        want = tuple(self.a.shape[:-1]) + (2 * self.a.shape[-1],)
        if tuple(self.u.shape) != want:
            raise StructuralError(f"Block2x2 u must have shape {want}, got {tuple(self.u.shape)}")

    @property
    def dim(self) -> int:
        return 2 * self.a.shape[-1]

    def nbytes(self) -> int:
        return sum(t.numel() * t.element_size() for t in (self.a, self.b, self.c, self.d, self.u))


def identity_element(like):
    if isinstance(like, DiagElements):
        return DiagElements(torch.ones_like(like.j), torch.zeros_like(like.u))
    if isinstance(like, DenseElements):
        eye = torch.eye(like.dim, dtype=like.J.dtype, device=like.J.device).expand(like.J.shape).clone()
        return DenseElements(eye, torch.zeros_like(like.u))
    if isinstance(like, Block2x2Elements):
        return Block2x2Elements(torch.ones_like(like.a), torch.zeros_like(like.b), torch.zeros_like(like.c),
                                torch.ones_like(like.d), torch.zeros_like(like.u))
    raise StructuralError(f"not an affine element: {type(like).__name__}")


def _check_pair(e2, e1):
    if type(e2) is not type(e1):
        raise StructuralError(f"variant mismatch: {type(e2).__name__} vs {type(e1).__name__}")
    if e2.dim != e1.dim:
        raise StructuralError(f"dimension mismatch: {e2.dim} vs {e1.dim}")


def compose(e2, e1):
    """x -> e2(e1(x)) = (J2 J1, J2 u1 + u2) (pscan.py:203-226)."""
    _check_pair(e2, e1)
    if isinstance(e2, DiagElements):
        return DiagElements(e2.j * e1.j, e2.j * e1.u + e2.u)
    if isinstance(e2, DenseElements):
        return DenseElements(e2.J @ e1.J, torch.einsum("...ij,...j->...i", e2.J, e1.u) + e2.u)
    D = e1.a.shape[-1]
    u1x, u1v = e1.u[..., :D], e1.u[..., D:]
    u = torch.cat([e2.a * u1x + e2.b * u1v + e2.u[..., :D], e2.c * u1x + e2.d * u1v + e2.u[..., D:]], dim=-1)
    return Block2x2Elements(e2.a * e1.a + e2.b * e1.c, e2.a * e1.b + e2.b * e1.d,
                            e2.c * e1.a + e2.d * e1.c, e2.c * e1.b + e2.d * e1.d, u)


def apply_element(e, s):
    s = _tensor(s, e.u)
    if isinstance(e, DiagElements):
        return e.j * s + e.u
    if isinstance(e, DenseElements):
        return torch.einsum("...ij,...j->...i", e.J, s) + e.u
    D = e.a.shape[-1]
    x, v = s[..., :D], s[..., D:]
    return torch.cat([e.a * x + e.b * v + e.u[..., :D], e.c * x + e.d * v + e.u[..., D:]], dim=-1)


def _row(e, t):
    if isinstance(e, DiagElements):
        return DiagElements(e.j[t], e.u[t])
    if isinstance(e, DenseElements):
        return DenseElements(e.J[t], e.u[t])
    return Block2x2Elements(e.a[t], e.b[t], e.c[t], e.d[t], e.u[t])


def _length(e) -> int:
    lead = tuple(e.u.shape[:-1])
    if len(lead) != 1:
        raise StructuralError(f"expected time-stacked elements, got batch shape {lead}")
    return lead[0]


def sequential_affine_solve(elements, s0):
    """Plain loop s_t = J_t s_{t-1} + u_t (pscan.py:258-266); test oracle only."""
    T = _length(elements)
    s = _tensor(s0, elements.u)
    out = torch.empty((T, s.shape[-1]), dtype=s.dtype, device=s.device)
    for t in range(T):
        s = apply_element(_row(elements, t), s)
        out[t] = s
    return out


def parallel_affine_solve(elements, s0, workers=None, chunk=None, stats=None, out=None):
    """All prefixes (e_t o ... o e_1)(s0) via the CUDA single-pass scans."""
    lib = _lib.load()
    T = _length(elements)
    if isinstance(elements, DiagElements):
        mode, D, ref = _lib.CS_MODE_DIAG, elements.dim, elements.j
        W = D
    elif isinstance(elements, DenseElements):
        mode, D, ref = _lib.CS_MODE_DENSE, elements.dim, elements.J
        W = D
    elif isinstance(elements, Block2x2Elements):
        mode, D, ref = _lib.CS_MODE_BLOCK, elements.a.shape[-1], elements.a
        W = 2 * D
    else:
        raise StructuralError(f"not an affine element: {type(elements).__name__}")
    s0 = _tensor(s0, ref).to(ref.dtype).contiguous()
    if tuple(s0.shape) != (W,):
        raise StructuralError(f"s0 must have shape ({W},), got {tuple(s0.shape)}")
    dt = _lib.dtype_code(ref.dtype)
    if out is None:
        out = torch.empty((T, W), dtype=ref.dtype, device=ref.device)
    ws_bytes = lib.cs_scan_workspace_bytes(mode, dt, T, D)
    ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=ref.device)
    st = _lib.stream_ptr()
    if mode == _lib.CS_MODE_DIAG:
        j, u = elements.j.contiguous(), elements.u.contiguous()
        rc = lib.cs_scan_diag(dt, _lib.ptr(j), _lib.ptr(u), _lib.ptr(s0), _lib.ptr(out), T, D, _lib.ptr(ws),
                              ws_bytes, st)
    elif mode == _lib.CS_MODE_DENSE:
        J, u = elements.J.contiguous(), elements.u.contiguous()
        rc = lib.cs_scan_dense(dt, _lib.ptr(J), _lib.ptr(u), _lib.ptr(s0), _lib.ptr(out), T, D, _lib.ptr(ws),
                               ws_bytes, st)
    else:
        a, b, c, d, u = (x.contiguous() for x in (elements.a, elements.b, elements.c, elements.d, elements.u))
        rc = lib.cs_scan_block(dt, _lib.ptr(a), _lib.ptr(b), _lib.ptr(c), _lib.ptr(d), _lib.ptr(u),
                               _lib.ptr(s0), _lib.ptr(out), T, D, _lib.ptr(ws), ws_bytes, st)
    _lib.check(rc)
    if stats is not None:
        n = ctypes.c_int(0)
        lib.cs_device_sm_count(ctypes.byref(n))
        stats.update(element_bytes=elements.nbytes(), scratch_bytes=int(ws_bytes),
                     output_bytes=out.numel() * out.element_size(), chunk=None, chunks=None,
                     workers=int(n.value))
    return out


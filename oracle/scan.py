"""Affine-scan algebra and the chunked parallel solve (TEST INFRASTRUCTURE ONLY).

Reference: ``chainscan/pscan.py``.  Element carriers (pscan.py:100-173), the
monoid (identity 176-191, compose 203-226, apply 229-240), the loop oracle
(258-266), the chunk policy (269-270) and the chunked two-pass solve
(273-354).  The chunked kernels are the C restatement in ``scan.c`` (built by
``oracle/Makefile`` into ``oracle/_build/liboracle_scan.so``).
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass

import numpy as np

from .errors import StructuralError

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle_scan.so")
_lib = None


def build_lib(force: bool = False) -> str:
    """Compile scan.c with gcc + OpenMP (no FMA contraction, like numba)."""
    if force or not os.path.exists(_LIB_PATH) or (
        os.path.getmtime(_LIB_PATH) < os.path.getmtime(os.path.join(_HERE, "scan.c"))
    ):
        subprocess.check_call(["make", "-s", "-C", _HERE])
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        build_lib()
        lib = ctypes.CDLL(_LIB_PATH)
        P = ctypes.POINTER(ctypes.c_double)
        i64 = ctypes.c_int64
        lib.oracle_scan_diag.argtypes = [P, P, P, i64, i64, i64, P]
        lib.oracle_scan_dense.argtypes = [P, P, P, i64, i64, i64, P]
        lib.oracle_scan_block.argtypes = [P, P, P, P, P, P, i64, i64, i64, P]
        lib.oracle_num_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def _ptr(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def workers_default() -> int:
    """CHAINSCAN_THREADS or the core count (pscan.py:50-62)."""
    raw = os.environ.get("CHAINSCAN_THREADS", "")
    try:
        n = int(raw)
        if n >= 1:
            return n
    except ValueError:
        pass
    return os.cpu_count() or 1


def _f64(x):
    return np.ascontiguousarray(np.asarray(x, dtype=np.float64))


@dataclass
class DiagElements:
    j: np.ndarray
    u: np.ndarray

    def __post_init__(self):
        self.j, self.u = _f64(self.j), _f64(self.u)
        if self.j.shape != self.u.shape:
            raise StructuralError("diag j/u shapes differ")

    @property
    def dim(self):
        return self.j.shape[-1]

    def nbytes(self):
        return self.j.nbytes + self.u.nbytes


@dataclass
class DenseElements:
    J: np.ndarray
    u: np.ndarray

    def __post_init__(self):
        self.J, self.u = _f64(self.J), _f64(self.u)
        if self.J.shape[-1] != self.J.shape[-2] or self.J.shape[:-1] != self.u.shape:
            raise StructuralError("dense J/u shapes inconsistent")

    @property
    def dim(self):
        return self.J.shape[-1]

    def nbytes(self):
        return self.J.nbytes + self.u.nbytes


@dataclass
class Block2x2Elements:
    a: np.ndarray
    b: np.ndarray
    c: np.ndarray
    d: np.ndarray
    u: np.ndarray

    def __post_init__(self):
        self.a, self.b, self.c, self.d, self.u = map(_f64, (self.a, self.b, self.c, self.d, self.u))
        for q in (self.b, self.c, self.d):
            if q.shape != self.a.shape:
                raise StructuralError("block diagonals must share a shape")
        if self.u.shape != self.a.shape[:-1] + (2 * self.a.shape[-1],):
            raise StructuralError("block u must be (..., 2D)")

    @property
    def dim(self):
        return 2 * self.a.shape[-1]

    def nbytes(self):
        return sum(x.nbytes for x in (self.a, self.b, self.c, self.d, self.u))


def identity_element(like):
    if isinstance(like, DiagElements):
        return DiagElements(np.ones_like(like.j), np.zeros_like(like.u))
    if isinstance(like, DenseElements):
        return DenseElements(np.broadcast_to(np.eye(like.dim), like.J.shape).copy(),
                             np.zeros_like(like.u))
    if isinstance(like, Block2x2Elements):
        one, zero = np.ones_like(like.a), np.zeros_like(like.a)
        return Block2x2Elements(one, zero, zero.copy(), one.copy(), np.zeros_like(like.u))
    raise StructuralError("not an affine element")


def compose(e2, e1):
    """x -> e2(e1(x)) = (J2 J1, J2 u1 + u2)."""
    if type(e2) is not type(e1) or e2.dim != e1.dim:
        raise StructuralError("variant or dimension mismatch")
    if isinstance(e2, DiagElements):
        return DiagElements(e2.j * e1.j, e2.j * e1.u + e2.u)
    if isinstance(e2, DenseElements):
        return DenseElements(e2.J @ e1.J, np.einsum("...ij,...j->...i", e2.J, e1.u) + e2.u)
    n = e1.a.shape[-1]
    x1, v1 = e1.u[..., :n], e1.u[..., n:]
    ux = e2.a * x1 + e2.b * v1 + e2.u[..., :n]
    uv = e2.c * x1 + e2.d * v1 + e2.u[..., n:]
    return Block2x2Elements(
        e2.a * e1.a + e2.b * e1.c,
        e2.a * e1.b + e2.b * e1.d,
        e2.c * e1.a + e2.d * e1.c,
        e2.c * e1.b + e2.d * e1.d,
        np.concatenate([ux, uv], axis=-1),
    )


def apply_element(e, s):
    s = np.asarray(s, dtype=np.float64)
    if isinstance(e, DiagElements):
        return e.j * s + e.u
    if isinstance(e, DenseElements):
        return np.einsum("...ij,...j->...i", e.J, s) + e.u
    n = e.a.shape[-1]
    x, v = s[..., :n], s[..., n:]
    return np.concatenate([e.a * x + e.b * v + e.u[..., :n],
                           e.c * x + e.d * v + e.u[..., n:]], axis=-1)


def _row(e, t):
    if isinstance(e, DiagElements):
        return DiagElements(e.j[t], e.u[t])
    if isinstance(e, DenseElements):
        return DenseElements(e.J[t], e.u[t])
    return Block2x2Elements(e.a[t], e.b[t], e.c[t], e.d[t], e.u[t])


def sequential_affine_solve(e, s0):
    """Loop s_t = J_t s_{t-1} + u_t (pscan.py:258-266)."""
    T = e.u.shape[0]
    s = np.asarray(s0, dtype=np.float64)
    out = np.empty((T, s.shape[-1]))
    for t in range(T):
        s = apply_element(_row(e, t), s)
        out[t] = s
    return out


def default_chunk(T: int, workers: int) -> int:
    """max(min(T, 256), ceil(T / (8 workers))) (pscan.py:269-270)."""
    return max(min(T, 256), math.ceil(T / (8 * workers)))


def parallel_affine_solve(e, s0, workers=None, chunk=None):
    """Chunked two-pass solve, bit-identical to the reference for equal chunk."""
    lib = _load()
    s0 = _f64(s0)
    if e.u.ndim != 2:
        raise StructuralError("expected time-stacked elements")
    T = e.u.shape[0]
    workers = workers_default() if workers is None else int(workers)
    chunk = default_chunk(T, workers) if chunk is None else int(chunk)
    chunk = max(1, min(chunk, T))
    if isinstance(e, DiagElements):
        D = e.dim
        if s0.shape != (D,):
            raise StructuralError("s0 shape")
        out = np.empty((T, D))
        lib.oracle_scan_diag(_ptr(e.j), _ptr(e.u), _ptr(s0), T, D, chunk, _ptr(out))
    elif isinstance(e, DenseElements):
        D = e.dim
        if s0.shape != (D,):
            raise StructuralError("s0 shape")
        out = np.empty((T, D))
        lib.oracle_scan_dense(_ptr(e.J), _ptr(e.u), _ptr(s0), T, D, chunk, _ptr(out))
    elif isinstance(e, Block2x2Elements):
        n = e.a.shape[-1]
        if s0.shape != (2 * n,):
            raise StructuralError("s0 shape")
        out = np.empty((T, 2 * n))
        lib.oracle_scan_block(_ptr(e.a), _ptr(e.b), _ptr(e.c), _ptr(e.d), _ptr(e.u),
                              _ptr(s0), T, n, chunk, _ptr(out))
    else:
        raise StructuralError("not an affine element")
    return out

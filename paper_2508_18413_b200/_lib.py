"""ctypes binding of libchainscan_b200.so (include/chainscan_b200.h).

The product path has no CPU fallback: if the library is missing or a CUDA
device is absent, calls raise.  Status codes map onto the reference's
exception types (chainscan/core.py:30-44, noise.py:30).
"""

from __future__ import annotations

import ctypes
import os

import torch

from .errors import ChainDivergedError, ConfigurationError, StructuralError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "libchainscan_b200.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "chainscan_b200.h")

CS_OK, CS_ERR_STRUCTURAL, CS_ERR_CONFIG, CS_ERR_DIVERGED, CS_ERR_CUDA, CS_ERR_INDEX = range(6)
CS_F32, CS_F64 = 0, 1
CS_NOISE_NORMAL, CS_NOISE_UNIFORM, CS_NOISE_CHI2, CS_NOISE_LOG_UNIFORM = range(4)
CS_TARGET_STD_NORMAL, CS_TARGET_GAUSSIAN, CS_TARGET_ROSENBROCK, CS_TARGET_MOG, CS_TARGET_BLR = range(5)
CS_SYS_MALA, CS_SYS_HMC, CS_SYS_LEAPFROG, CS_SYS_GIBBS = range(4)
CS_MODE_DENSE, CS_MODE_DIAG, CS_MODE_BLOCK = range(3)
CS_RUN_MAXITERS, CS_RUN_CONVERGED, CS_RUN_DIVERGED = range(3)
CS_DIV_NONE, CS_DIV_PROPOSAL, CS_DIV_STEP, CS_DIV_JACOBIAN, CS_DIV_GUARD = range(5)
CS_STOP_MAXITERS, CS_STOP_PICARD, CS_STOP_NOFAIL, CS_STOP_ERROR = range(4)

P = ctypes.c_void_p
i32, i64, u64, f64, szt = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double, ctypes.c_size_t


class cs_target(ctypes.Structure):
    _fields_ = [("kind", i32), ("dim", i32), ("a", f64), ("b", f64), ("scale1", f64),
                ("scale2", f64), ("mu", P), ("chol", P), ("prec", P), ("n_comp", i32),
                ("means", P), ("variances", P), ("logw", P), ("lognorm", P),
                ("n_data", i64), ("X", P), ("y", P), ("prior_precision", f64)]


class cs_system(ctypes.Structure):
    _fields_ = [("kind", i32), ("dim", i32), ("target", cs_target), ("eps", f64), ("L", i32),
                ("mass", P), ("seed", u64), ("probe_seed", u64), ("T", i64),
                ("noise_vec", P), ("noise_logu", P), ("g_tau", P), ("xi_mu", P),
                ("xi_theta", P), ("g_sigma", P), ("gibbs", P), ("basis", P)]


class cs_deer_config(ctypes.Structure):
    _fields_ = [("mode", i32), ("atol", f64), ("rtol", f64), ("max_iters", i32),
                ("hutchinson_samples", i32), ("damping", f64), ("clip", f64),
                ("preconditioner", P)]


class cs_deer_result(ctypes.Structure):
    _fields_ = [("iterations", i32), ("status", i32), ("err_kind", i32), ("err_step", i64),
                ("err_iteration", i32), ("launches", i32), ("guard_dmax", f64),
                ("guard_d0", f64), ("stop_reason", i32), ("grid_blocks", i32),
                ("steps_per_thread", i32), ("kept_in_registers", i32), ("fused_tangent", i32),
                ("device_ms", f64)]


class cs_elem_stats(ctypes.Structure):
    _fields_ = [("bad_proposal", i64), ("bad_step", i64), ("bad_jacobian", i64), ("picard_fail", ctypes.c_uint32),
                ("fail_rows", ctypes.c_uint32), ("dmax", f64)]


SP = ctypes.POINTER(cs_system)
CP = ctypes.POINTER(cs_deer_config)
_SIGS = {
    "cs_last_error": ([], ctypes.c_char_p),
    "cs_version": ([], ctypes.c_int),
    "cs_debug_probe": ([P, ctypes.c_int], ctypes.c_int),
    "cs_debug_gram": ([P, i32, i32, P, i64, P, P], ctypes.c_int),
    "cs_debug_pair_gram": ([P, i32, i32, P, i64, P, P], ctypes.c_int),
    "cs_device_sm_count": ([ctypes.POINTER(ctypes.c_int)], ctypes.c_int),
    "cs_stream_sync": ([P], ctypes.c_int),
    "cs_target_eval": ([ctypes.POINTER(cs_target), ctypes.c_int, i64, P, P, P, P], ctypes.c_int),
    "cs_noise_fill": ([ctypes.c_int, u64, u64, i64, i64, i32, f64, ctypes.c_int, P, P], ctypes.c_int),
    "cs_rademacher_fill": ([u64, i64, P, i64, i64, i32, i32, ctypes.c_int, P, P], ctypes.c_int),
    "cs_scan_workspace_bytes": ([ctypes.c_int, ctypes.c_int, i64, i32], szt),
    "cs_scan_diag": ([ctypes.c_int, P, P, P, P, i64, i32, P, szt, P], ctypes.c_int),
    "cs_scan_block": ([ctypes.c_int, P, P, P, P, P, P, P, i64, i32, P, szt, P], ctypes.c_int),
    "cs_scan_dense": ([ctypes.c_int, P, P, P, P, i64, i32, P, szt, P], ctypes.c_int),
    "cs_scan_aggregate": ([ctypes.c_int, ctypes.c_int, P, P, P, P, P, i64, i32, P, P, szt, P], ctypes.c_int),
    "cs_first_nonfinite_row": ([ctypes.c_int, P, i64, i64, P, P], ctypes.c_int),
    "cs_first_stamped_row": ([P, i64, i32, P, P], ctypes.c_int),
    "cs_converged": ([ctypes.c_int, P, P, i64, f64, f64, P, P, P], ctypes.c_int),
    "cs_update_bookkeeping": ([ctypes.c_int, P, P, i64, i32, f64, f64, i32, P, P, P, P], ctypes.c_int),
    "cs_form_diag": ([ctypes.c_int, P, P, P, P, i64, i32, P, f64, f64, P, P, P], ctypes.c_int),
    "cs_form_dense": ([ctypes.c_int, P, P, P, P, i64, i32, P, f64, f64, P, P, P], ctypes.c_int),
    "cs_form_block": ([ctypes.c_int, P, P, P, P, P, P, P, i64, i32, P, f64, f64, P, P, P, P, P, P],
                      ctypes.c_int),
    "cs_hutchinson_accumulate": ([ctypes.c_int, P, P, P, i64, i32, f64, P], ctypes.c_int),
    "cs_system_supported": ([SP, ctypes.c_int], ctypes.c_int),
    "cs_system_step": ([SP, ctypes.c_int, P, i64, i64, P, P, P, P], ctypes.c_int),
    "cs_system_jvp": ([SP, ctypes.c_int, P, i64, i64, P, P, P, i32, P], ctypes.c_int),
    "cs_system_relaxed_step": ([SP, ctypes.c_int, P, i64, i64, P, P, P], ctypes.c_int),
    "cs_system_block_jacobian": ([SP, ctypes.c_int, P, i64, i64, P, i32, i64, P, P, P, P, P],
                                 ctypes.c_int),
    "cs_system_sequential": ([SP, ctypes.c_int, P, i64, P, P, P], ctypes.c_int),
    "cs_system_elements": ([SP, CP, ctypes.c_int, i64, P, P, P, P, P, P, P, P, P], ctypes.c_int),
    "cs_system_elements_range": ([SP, CP, ctypes.c_int, i64, i64, i64, P, P, P, P, P, P, P, P, P], ctypes.c_int),
    "cs_system_elements_supported": ([SP, i32, ctypes.c_int], ctypes.c_int),
    "cs_system_elements_range_supported": ([SP, CP, ctypes.c_int], ctypes.c_int),
    "cs_scan_diag_update": ([ctypes.c_int, P, P, P, P, i64, i32, P, szt, P, f64, f64, i32, P, P, P], ctypes.c_int),
    "cs_scan_block_update": ([ctypes.c_int, P, P, P, P, P, P, P, i64, i32, P, szt, P, f64, f64, i32, P, P, P],
                             ctypes.c_int),
    "cs_deer_workspace_bytes": ([SP, ctypes.c_int, i32], szt),
    "cs_leapfrog_batch_supported": ([SP, i32, ctypes.c_int], ctypes.c_int),
    "cs_leapfrog_batch_solve": ([SP, ctypes.POINTER(cs_deer_config), ctypes.c_int, i32, P, P, P, P, P], ctypes.c_int),
    "cs_deer_supported": ([SP, ctypes.c_int, ctypes.c_int], ctypes.c_int),
    "cs_deer_solve": ([SP, ctypes.POINTER(cs_deer_config), ctypes.c_int, P, P, P, P, P, szt,
                       ctypes.POINTER(cs_deer_result), P], ctypes.c_int),
}

_lib = None


def load():
    """Load the CUDA library; raise loudly if it is missing (no fallback)."""
    global _lib
    if _lib is None:
        # tuning experiments only: a variant build of the same library
        LIB_PATH_ = os.environ.get("CS_LIB_PATH", LIB_PATH)
        if LIB_PATH_ != LIB_PATH:
            return _load_path(LIB_PATH_)
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"libchainscan_b200.so not found at {LIB_PATH}; build it with "
                "`python -m paper_2508_18413_b200.build` (there is no CPU fallback)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (args, res) in _SIGS.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        _lib = lib
    return _lib


def _load_path(path):
    global _lib
    lib = ctypes.CDLL(path)
    for name, (args, res) in _SIGS.items():
        fn = getattr(lib, name, None)  # an older variant may predate an entry point
        if fn is None:
            continue
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return _lib


def exported_symbols():
    return sorted(_SIGS)


def check(rc: int, step=None, iteration=None):
    if rc == CS_OK:
        return
    msg = load().cs_last_error().decode()
    if rc == CS_ERR_STRUCTURAL:
        raise StructuralError(msg)
    if rc == CS_ERR_CONFIG:
        raise ConfigurationError(msg)
    if rc == CS_ERR_DIVERGED:
        raise ChainDivergedError(msg, step=step, iteration=iteration)
    if rc == CS_ERR_INDEX:
        raise IndexError(msg)
    raise RuntimeError(f"CUDA error: {msg}")


def require_cuda():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2508_18413_b200 needs a CUDA device (B200); no CPU fallback")


_RAW_STREAM = getattr(torch._C, "_cuda_getCurrentRawStream", None)
_CUR_DEVICE = getattr(torch._C, "_cuda_getDevice", None)


def stream_ptr(stream=None):
    # the current stream's raw handle without building a torch.cuda.Stream
    # object (15 us per call through torch.cuda.current_stream()); the public
    # path when this torch build lacks the private accessors
    if stream is not None:
        return ctypes.c_void_p(stream.cuda_stream)
    if _RAW_STREAM is not None and _CUR_DEVICE is not None:
        return ctypes.c_void_p(_RAW_STREAM(_CUR_DEVICE()))
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def sync_current():
    """Synchronise the current stream of the current device (cheaper than
    torch.cuda.current_stream().synchronize())."""
    check(load().cs_stream_sync(stream_ptr()))


def ptr(t):
    return ctypes.c_void_p(0 if t is None else t.data_ptr())


def dtype_code(dtype):
    if dtype == torch.float32:
        return CS_F32
    if dtype == torch.float64:
        return CS_F64
    raise ConfigurationError(f"unsupported dtype {dtype}; use torch.float32 or torch.float64")

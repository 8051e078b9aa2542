"""Python-side cost of the pieces of run_deer's fused path (development)."""
import os, sys, time, ctypes
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_18413_b200 as cs
from paper_2508_18413_b200 import _lib, deer
m = cs.model_logp_grad_hvp(cs.rosenbrock(a=0.0, b=0.1, scale1=1.0, scale2=1.0))
k = cs.HmcKernel(m, 0.5, 8, seed=0, T=100_000, dtype=torch.float32)
cfg = cs.DeerConfig(mode="diag-stochastic", clip=1.0)
s0 = torch.zeros(2, dtype=torch.float32, device="cuda")
for _ in range(5): cs.run_deer(k, s0, cfg)
torch.cuda.synchronize()
def t(name, fn, n=2000):
    fn()
    t0 = time.perf_counter_ns()
    for _ in range(n): fn()
    print(f"{name:40s} {(time.perf_counter_ns() - t0) / n / 1e3:7.2f} us")
t("as_tensor+contiguous", lambda: torch.as_tensor(s0, dtype=k.dtype, device=k.device).contiguous())
t("_pre_tensor", lambda: deer._pre_tensor(cfg, k.device, k.dim))
t("default_max_iters", lambda: deer.default_max_iters(k.T))
t("_pick_engine", lambda: deer._pick_engine(k, cfg))
t("desc()", lambda: k.desc())
t("torch.empty trace", lambda: torch.empty((100_000, 2), dtype=torch.float32, device="cuda"))
t("torch.empty psca", lambda: torch.empty(100_000, dtype=torch.int32, device="cuda"))
t("_pinned_hist", lambda: deer._pinned_hist(400))
t("cs_deer_result()", lambda: _lib.cs_deer_result())
t("stream_ptr", lambda: _lib.stream_ptr())
t("ptr x5", lambda: [_lib.ptr(s0) for _ in range(5)])
hist = deer._pinned_hist(400)
t("hist[:14].numpy().copy()", lambda: hist[:14].numpy().copy())
t("DeerResult(...)", lambda: deer.DeerResult(trace=s0, iterations=14, delta_history=None, converged=True,
                                             per_step_converged_at=s0, full_trace=None, stats={}))
t("key tuple", lambda: (cfg.mode, k.dtype, 400, cfg.atol, cfg.rtol, cfg.hutchinson_samples, cfg.damping, cfg.clip,
                         None if cfg.preconditioner is None else cfg.preconditioner.tobytes(), k.T, k.device))
# whole calls
t("run_deer (fused, full solve)", lambda: cs.run_deer(k, s0, cfg), n=300)
d = k.desc()
c = k._fused_ws[next(iter(k._fused_ws))][3]
lib = _lib.load()
tr = torch.empty((100_000, 2), dtype=torch.float32, device="cuda")
ps = torch.empty(100_000, dtype=torch.int32, device="cuda")
ws, wsb = k._fused_ws[next(iter(k._fused_ws))][0], k._fused_ws[next(iter(k._fused_ws))][1]


def raw():
    res = _lib.cs_deer_result()
    lib.cs_deer_solve(ctypes.byref(d), ctypes.byref(c), _lib.dtype_code(k.dtype), _lib.ptr(s0), _lib.ptr(tr),
                      _lib.ptr(ps), _lib.ptr(hist), _lib.ptr(ws), wsb, ctypes.byref(res), _lib.stream_ptr())


t("cs_deer_solve via ctypes only", raw, n=300)

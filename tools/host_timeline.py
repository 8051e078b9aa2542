"""Host-side timeline of one headline solve (development): Python prelude, the
C call (launch + device + sync), Python epilogue, against the bench's event
bracket."""
import ctypes
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_18413_b200 as cs  # noqa: E402
from paper_2508_18413_b200 import _lib  # noqa: E402

m = cs.model_logp_grad_hvp(cs.rosenbrock(a=0.0, b=0.1, scale1=1.0, scale2=1.0))
k = cs.HmcKernel(m, 0.5, 8, seed=0, T=100_000, dtype=torch.float32)
cfg = cs.DeerConfig(mode="diag-stochastic", clip=1.0)
s0 = torch.zeros(2, dtype=torch.float32, device="cuda")
for _ in range(10):
    r = cs.run_deer(k, s0, cfg)
torch.cuda.synchronize()
lib = _lib.load()
ws, ws_bytes, pre, c = next(iter(k._fused_ws.values()))
d = k.desc()
trace = torch.empty((100_000, 2), device="cuda")
psca = torch.empty(100_000, dtype=torch.int32, device="cuda")
hist = torch.empty(400, dtype=torch.float64).pin_memory()
res = _lib.cs_deer_result()
sp = _lib.stream_ptr()
args = (ctypes.byref(d), ctypes.byref(c), _lib.dtype_code(torch.float32), _lib.ptr(s0), _lib.ptr(trace), _lib.ptr(psca),
        _lib.ptr(hist), _lib.ptr(ws), ws_bytes, ctypes.byref(res), sp)
for _ in range(5):
    lib.cs_deer_solve(*args)
walls, dev = [], []
for _ in range(100):
    t0 = time.perf_counter_ns()
    lib.cs_deer_solve(*args)
    walls.append((time.perf_counter_ns() - t0) / 1e3)
    dev.append(res.device_ms * 1e3)
print(f"bare C call: wall {np.median(walls):.1f} us, device_ms {np.median(dev):.1f} us")
# event bracket around the bare call and around run_deer
for name, fn in (("bare", lambda: lib.cs_deer_solve(*args)), ("run_deer", lambda: cs.run_deer(k, s0, cfg))):
    ts = []
    for _ in range(50):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    print(f"event bracket {name}: {np.median(ts):.1f} us")
t = []
for _ in range(200):
    t0 = time.perf_counter_ns()
    cs.run_deer(k, s0, cfg)
    t.append((time.perf_counter_ns() - t0) / 1e3)
print(f"run_deer wall {np.median(t):.1f} us")
# the kernel alone (ncu-free): back-to-back launches without host work between

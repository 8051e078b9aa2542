"""HMC 2D standard normal at T = 2^20 (streamed engine: element kernel + fused-bookkeeping
diag scan at D = 2 per iteration); development probe for the small-D update scan."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_18413_b200 as cs  # noqa: E402

m = cs.model_logp_grad_hvp(cs.std_normal(2))
k = cs.HmcKernel(m, 0.5, 8, seed=0, T=1 << 20, dtype=torch.float32)
cfg = cs.DeerConfig(mode="diag-stochastic", clip=1.0)
s0 = torch.zeros(2, dtype=torch.float32, device="cuda")
r = cs.run_deer(k, s0, cfg)
ts = []
for _ in range(5):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    r2 = cs.run_deer(k, s0, cfg)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
print(f"T=2^20 HMC 2D std-normal streamed: {np.median(ts):.3f} ms, {r2.iterations} iterations, path {r2.stats.get('path')}, "
      f"trace checksum {float(r2.trace.double().sum()):.6f}")

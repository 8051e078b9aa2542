"""Diag / block row-scan throughput at HBM-sized T (development sweep; env
CS_SCAN_ROUND_KB / CS_SCAN_LAG select the carry-scan geometry)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_18413_b200 as cs  # noqa: E402

kind = sys.argv[1] if len(sys.argv) > 1 else "diag"
T = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 24
D = int(sys.argv[3]) if len(sys.argv) > 3 else 18
dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(0)
s0 = torch.zeros(D if kind == "diag" else 2 * D, device=dev)
if kind == "diag":
    el = cs.DiagElements((torch.rand((T, D), generator=g, device=dev) * 1.8 - 0.9), torch.randn((T, D), generator=g, device=dev))
    byts = 12 * T * D
    out = torch.empty((T, D), device=dev)
else:
    el = cs.Block2x2Elements(*[(torch.rand((T, D), generator=g, device=dev) * 1.2 - 0.6) for _ in range(4)],
                             torch.randn((T, 2 * D), generator=g, device=dev))
    byts = 32 * T * D
    out = torch.empty((T, 2 * D), device=dev)
for _ in range(3):
    cs.parallel_affine_solve(el, s0, out=out)
ref = out.clone()
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
ts = []
for _ in range(10):
    flush.fill_(0.0)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    cs.parallel_affine_solve(el, s0, out=out)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
ms = float(np.median(ts))
print(f"{kind} T={T} D={D} round_kb={os.environ.get('CS_SCAN_ROUND_KB', 'dflt')} lag={os.environ.get('CS_SCAN_LAG', 'dflt')}: "
      f"{ms:.3f} ms  {byts / ms / 1e6:.0f} GB/s  ({byts / ms / 1e6 / 6551.7:.1%} of HBM)  identical={bool(torch.equal(out, ref))}", flush=True)

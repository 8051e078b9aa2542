"""Per-phase timing of the persistent solver via cs_debug_probe (development)."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_18413_b200 as cs  # noqa: E402
from paper_2508_18413_b200 import _lib  # noqa: E402
from probe_solve import make  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "hmc"
T = int(sys.argv[2]) if len(sys.argv) > 2 else 100_000
k, s0, cfg = make(cfgname, T, torch.float32)
cfg.engine = "fused"
cs.run_deer(k, s0, cfg)
buf = torch.zeros(64 * 8, dtype=torch.int64, device="cuda")
_lib.load().cs_debug_probe(ctypes.c_void_p(buf.data_ptr()), 64 * 8)
r = cs.run_deer(k, s0, cfg)
torch.cuda.synchronize()
_lib.load().cs_debug_probe(ctypes.c_void_p(0), 0)
t = buf.cpu().numpy().reshape(64, 8).astype(np.float64)
names = ["halo", "phaseA", "blkscan+flags", "gridsync", "decide+fold", "replay", "->next"]
print(f"{cfgname} T={T} iters={r.iterations} stats={r.stats}")
for it in range(min(r.iterations + 1, 20)):
    row = t[it]
    d = []
    for kk in range(6):
        d.append((row[kk + 1] - row[kk]) / 1e3 if row[kk + 1] and row[kk] else float("nan"))
    nxt = (t[it + 1][0] - row[6]) / 1e3 if t[it + 1][0] and row[6] else float("nan")
    print(f"it {it:2d}: " + "  ".join(f"{n}={v:6.2f}" for n, v in zip(names, d + [nxt])) + " us")

"""cfg 5 through run_deer_sharded on an NCCL group of one vs the single-GPU engine (development)."""
import os
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_18413_b200 as cs  # noqa: E402
from paper_2508_18413_b200.sharded import run_deer_sharded  # noqa: E402

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29561")
dist.init_process_group("nccl", device_id=torch.device("cuda", 0), rank=0, world_size=1)
k = cs.GibbsKernel(cs.generate_eight_schools(), seed=0, T=1_000_000, dtype=torch.float32)
cfg = cs.DeerConfig(mode="diag-stochastic", hutchinson_samples=3, preconditioner=k.recommended_preconditioner(),
                    max_iters=400)
s0 = k.initial_state()
for name, fn in (("sharded (NCCL x1)", lambda: run_deer_sharded(k, s0, cfg)), ("run_deer", lambda: cs.run_deer(k, s0, cfg))):
    fn()
    ts = []
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    print(f"{name}: {1e3 * np.median(ts):.1f} ms, iterations {r.iterations}", flush=True)
dist.destroy_process_group()

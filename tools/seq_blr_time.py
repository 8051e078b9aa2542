"""Time the device sequential walk of cfg 3's BLR MALA chain (development)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_18413_b200 as cs  # noqa: E402

X, y, _ = cs.synthetic_credit_like(seed=20250819, n=1000, dim=100)
k = cs.MalaKernel(cs.model_logp_grad_hvp(cs.blr(X, y, 1.0)), 0.003, seed=4, T=100_000)
for T in (1000, 100_000):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = cs.sequential_evaluate(k, np.zeros(100), T)
    torch.cuda.synchronize()
    print(f"BLR sequential walk T={T}: {time.perf_counter() - t0:.3f} s", flush=True)
g = np.load(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests/golden/big_cfg3_mala_blr100_T100K.npz"))
seq = out.cpu().numpy()
print("max |seq - reference seq rows|", float(np.max(np.abs(seq[499::500] - g["seq_rows"]))),
      "last", float(np.max(np.abs(seq[-1] - g["seq_last"]))))
acc = np.any(np.diff(np.vstack([np.zeros(100), seq]), axis=0) != 0, axis=1)
ref = np.unpackbits(g["seq_accept_bits"])[:100_000].astype(bool)
print("accept mask identical:", bool(np.array_equal(acc, ref)), "acceptance", acc.mean())

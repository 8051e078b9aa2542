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
NB = 1024 + 8 * 1024
buf = torch.zeros(NB, dtype=torch.int64, device="cuda")
_lib.load().cs_debug_probe(ctypes.c_void_p(buf.data_ptr()), NB)
r = cs.run_deer(k, s0, cfg)
torch.cuda.synchronize()
_lib.load().cs_debug_probe(ctypes.c_void_p(0), 0)
allb = buf.cpu().numpy().astype(np.float64)
t = allb[:512].reshape(64, 8)
names = ["halo", "phaseA", "blkscan+flags", "gridsync", "decide+fold", "replay", "->next"]
print(f"{cfgname} T={T} iters={r.iterations} stats={r.stats}")
for it in range(min(r.iterations + 1, 20)):
    row = t[it]
    d = []
    for kk in range(6):
        d.append((row[kk + 1] - row[kk]) / 1e3 if row[kk + 1] and row[kk] else float("nan"))
    nxt = (t[it + 1][0] - row[6]) / 1e3 if t[it + 1][0] and row[6] else float("nan")
    print(f"it {it:2d}: " + "  ".join(f"{n}={v:6.2f}" for n, v in zip(names, d + [nxt])) + " us")

# skew across CTAs in iteration 4: phase-A start (k=1), barrier arrival (k=3), exit (k=4)
cta = allb[1024:].reshape(-1, 8)
cta = cta[cta[:, 1] > 0]
if len(cta):
    t0 = cta[:, 1].min()
    st, ar, ex = (cta[:, 1] - t0) / 1e3, (cta[:, 3] - t0) / 1e3, (cta[:, 4] - t0) / 1e3
    pa = ar - st
    print(f"iteration 4 over {len(cta)} CTAs: phaseA+blkscan per CTA p10/50/90/max = "
          + " ".join(f"{v:.2f}" for v in np.percentile(pa, [10, 50, 90, 100])) + " us")
    print(f"  start skew max-min = {st.max() - st.min():.2f} us; arrival spread = {ar.max() - ar.min():.2f} us; "
          f"exit spread = {ex.max() - ex.min():.2f} us; last arrival -> first exit = {ex.min() - ar.max():.2f} us")

    fo, rp = (cta[:, 5] - cta[:, 4]) / 1e3, (cta[:, 6] - cta[:, 5]) / 1e3
    en = (cta[:, 6] - t0) / 1e3
    q = lambda x: " ".join(f"{v:.2f}" for v in np.percentile(x, [10, 50, 90, 100]))
    print(f"  decide+fold p10/50/90/max = {q(fo)} us;  replay+flags = {q(rp)} us; end spread = {en.max() - en.min():.2f} us")
    order = np.argsort(en)
    print("  latest-ending CTAs:", [int(i) for i in order[-8:]], " earliest:", [int(i) for i in order[:8]])

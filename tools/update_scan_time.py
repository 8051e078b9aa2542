"""Time the fused-bookkeeping update scan (cs_scan_diag_update) at one shape:
python tools/update_scan_time.py T D [slow]  (env CS_SCAN_RR picks the kernel)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_18413_b200 import _lib  # noqa: E402

T, D = int(sys.argv[1]), int(sys.argv[2])
slow = len(sys.argv) > 3 and sys.argv[3] == "slow"
lib = _lib.load()
dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(0)
j = (torch.rand((T, D), generator=g, device=dev) * (0.0009 if slow else 1.8) + (0.999 if slow else -0.9)).float()
u = torch.randn((T, D), generator=g, device=dev) * 1e-3
s0 = torch.zeros(D, device=dev)
guess = torch.randn((T, D), generator=g, device=dev)
out = torch.empty_like(guess)
lf = torch.zeros(T, dtype=torch.int32, device=dev)
st = torch.zeros(40, dtype=torch.uint8, device=dev)
wsb = lib.cs_scan_workspace_bytes(_lib.CS_MODE_DIAG, _lib.CS_F32, T, D)
ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)


def run():
    _lib.check(lib.cs_scan_diag_update(_lib.CS_F32, _lib.ptr(j), _lib.ptr(u), _lib.ptr(s0), _lib.ptr(out), T, D,
                                       _lib.ptr(ws), wsb, _lib.ptr(guess), 1e-5, 1e-5, 3, _lib.ptr(lf), _lib.ptr(st),
                                       _lib.stream_ptr()))


for _ in range(3):
    run()
ts = []
for _ in range(10):
    flush.fill_(0.0)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    run()
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
ms = float(np.median(ts))
print(f"update scan T={T} D={D} {'slow' if slow else 'fast'} CS_SCAN_RR={os.environ.get('CS_SCAN_RR', '2')}: {ms:.3f} ms "
      f"({20 * T * D / ms / 1e6:.0f} GB/s at 20 B/element)", flush=True)

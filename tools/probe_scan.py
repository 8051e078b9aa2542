"""Time the standalone affine scans at HBM-sized problems (development probe)."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_18413_b200 as cs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mode", default="diag")
    ap.add_argument("--T", type=int, default=1 << 22)
    ap.add_argument("--D", type=int, default=18)
    ap.add_argument("--dtype", default="f32")
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    dt = torch.float32 if a.dtype == "f32" else torch.float64
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(0)
    T, D = a.T, a.D
    es = 4 if dt == torch.float32 else 8
    if a.mode == "diag":
        el = cs.DiagElements((torch.rand((T, D), generator=g, device=dev) * 1.8 - 0.9).to(dt),
                             torch.randn((T, D), generator=g, device=dev).to(dt))
        s0 = torch.zeros(D, device=dev, dtype=dt)
        byts = 3 * T * D * es
    else:
        el = cs.Block2x2Elements(*[(torch.rand((T, D), generator=g, device=dev) * 1.2 - 0.6).to(dt) for _ in range(4)],
                                 torch.randn((T, 2 * D), generator=g, device=dev).to(dt))
        s0 = torch.zeros(2 * D, device=dev, dtype=dt)
        byts = 8 * T * D * es
    out = cs.parallel_affine_solve(el, s0)
    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
    ts = []
    for _ in range(a.reps):
        flush.fill_(0.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        cs.parallel_affine_solve(el, s0, out=out)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = float(np.median(ts))
    print(f"{a.mode} T={T} D={D} {a.dtype}: {ms:.3f} ms  {byts / ms / 1e6:.1f} GB/s (algorithmic {byts / 1e6:.0f} MB)")


if __name__ == "__main__":
    main()

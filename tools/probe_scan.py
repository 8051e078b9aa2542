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
    ap.add_argument("--trace", action="store_true", help="per-tile phase timeline (cs_debug_probe)")
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
    if a.trace:
        from paper_2508_18413_b200 import _lib
        n = min(T, 1 << 20)
        buf = torch.zeros(n * 16, dtype=torch.int64, device=dev)
        _lib.load().cs_debug_probe(buf.data_ptr(), buf.numel())
        flush.fill_(0.0)
        torch.cuda.synchronize()
        cs.parallel_affine_solve(el, s0, out=out)
        torch.cuda.synchronize()
        _lib.load().cs_debug_probe(None, 0)
        tr = buf.view(-1, 16).cpu().numpy().astype(np.int64)
        idx = np.nonzero(tr[:, 1] > 0)[0]
        tr = tr[idx]
        nt = len(tr)
        t0 = tr[:, 1].min()
        st = {k: tr[:, k] - t0 for k in range(1, 10)}
        span = st[9].max()
        q = lambda x: " ".join(f"{v / 1e3:7.2f}" for v in np.percentile(x, [10, 50, 90, 99]))
        print(f"tiles={nt} span={span / 1e3:.1f}us; steady state = tiles claimed in the middle half (us, p10/50/90/99)")
        inflight = [int(np.sum((st[1] <= t) & (st[9] > t))) for t in np.linspace(span * 0.2, span * 0.8, 7)]
        print(f"  tiles in flight: {inflight}; SMs used: {np.unique(tr[:, 0]).size}")
        m = (st[1] > 0.25 * span) & (st[1] < 0.75 * span)
        print(f"  claims per us (steady): {m.sum() / (0.5 * span / 1e3):.1f}")
        names = {1: "claim", 2: "p.start", 3: "p.reduced", 4: "p.published", 5: "c.start", 6: "c.ingroup",
                 7: "c.groups", 8: "c.entry", 9: "c.store"}
        for k0, k1 in ((1, 2), (2, 3), (3, 4), (4, 5), (5, 6), (5, 7), (7, 8), (8, 9), (1, 9)):
            print(f"  {names[k0]:>11s}->{names[k1]:<11s} {q((st[k1] - st[k0])[m])}")


if __name__ == "__main__":
    main()

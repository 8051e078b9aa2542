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
    ap.add_argument("--agg", action="store_true", help="also time the aggregate-only (reduce) pass")
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
    elif a.mode == "dense":
        el = cs.DenseElements((torch.randn((T, D, D), generator=g, device=dev) * (0.45 / D ** 0.5)).to(dt),
                              torch.randn((T, D), generator=g, device=dev).to(dt))
        s0 = torch.zeros(D, device=dev, dtype=dt)
        byts = T * (D * D + 2 * D) * es
        print(f"  dense: {2 * T * D ** 3 / 1e9:.1f} GFLOP of composition")
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
    if a.agg and a.mode == "diag":
        from paper_2508_18413_b200 import _lib
        lib = _lib.load()
        dtc = 1 if dt == torch.float64 else 0
        wsb = lib.cs_scan_workspace_bytes(1, dtc, T, D)
        ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev)
        agg = torch.empty(2 * D, dtype=torch.float64, device=dev)
        ta = []
        for _ in range(a.reps):
            flush.fill_(0.0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            lib.cs_scan_aggregate(1, dtc, el.j.data_ptr(), None, None, None, el.u.data_ptr(), T, D, agg.data_ptr(),
                                  ws.data_ptr(), wsb, None)
            e1.record()
            torch.cuda.synchronize()
            ta.append(e0.elapsed_time(e1))
        ma = float(np.median(ta))
        print(f"  aggregate-only: {ma:.3f} ms  {2 * T * D * es / ma / 1e6:.1f} GB/s read")
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
        idx = np.nonzero(tr[:, 4] > 0)[0]
        tr = tr[idx]
        nt = len(tr)
        t0 = tr[:, 4].min()
        st = {k: tr[:, k] - t0 for k in range(1, 15)}
        span = st[9].max()
        q = lambda x: " ".join(f"{v / 1e3:7.2f}" for v in np.percentile(x, [10, 50, 90, 99]))
        print(f"chunks={nt} span={span / 1e3:.1f}us (us, p10/50/90/99 over the middle half)")
        m = (st[4] > 0.25 * span) & (st[4] < 0.75 * span)
        lbw = os.environ.get("CS_SCAN_LBW", "1") != "0"
        if lbw:  # look-back warp: 6/7 = its lookup start/end
            names = {4: "A.published", 5: "C.start", 6: "LB.start", 7: "LB.end", 8: "C.entry", 9: "C.laststore"}
            names.update({10: "LB.gpoll", 11: "LB.gfold", 12: "LB.exit", 13: "LB.ipoll", 14: "LB.ifold",
                          1: "A.start", 2: "A.end", 3: "P.groupdone"})
            pairs = ((1, 2), (2, 4), (4, 3), (2, 5), (4, 5), (4, 6), (6, 7), (6, 10), (10, 11), (11, 12), (12, 13), (13, 14), (14, 7), (7, 8),
                     (5, 8), (8, 9))
        else:
            names = {4: "A.published", 5: "C.start", 6: "C.ingroup", 7: "C.groups", 8: "C.entry", 9: "C.laststore"}
            pairs = ((4, 5), (5, 6), (5, 7), (7, 8), (5, 8), (8, 9))
        if lbw and os.environ.get("CS_TRACE_CTA"):
            # one CTA's event sequence (chunks j, j+G, ...; G = grid size)
            G = int(os.environ.get("CS_TRACE_G", "444"))
            j = int(os.environ["CS_TRACE_CTA"])
            ev = []
            full = buf.view(-1, 16).cpu().numpy().astype(np.int64)
            for q in range(j, min(len(full), j + 12 * G), G):
                for k in (1, 2, 4, 3, 6, 10, 11, 13, 14, 7, 5, 8, 9):
                    if full[q, k] > 0:
                        ev.append((full[q, k], q // G, names.get(k, str(k))))
            ev.sort()
            e0 = ev[0][0]
            print("  ".join(f"{(t - e0) / 1e3:.1f}:{nm}@{r}" for t, r, nm in ev))
        for k0, k1 in pairs:
            print(f"  {names[k0]:>11s}->{names[k1]:<11s} {q((st[k1] - st[k0])[m])}")


if __name__ == "__main__":
    main()

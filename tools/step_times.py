import os, sys, gc, json
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import bench
import paper_2508_18413_b200 as cs
dev = torch.device("cuda")
m = cs.model_logp_grad_hvp(cs.rosenbrock(**bench.ROSEN))
k = cs.HmcKernel(m, bench.EPS, bench.LSTEPS, seed=0, T=100_000, dtype=torch.float32)
cfg = cs.DeerConfig(mode="diag-stochastic", clip=1.0)
s0 = torch.zeros(2, device=dev)
flush = torch.empty(256 * 1024 * 1024 // 4, device=dev)
for _ in range(5): cs.run_deer(k, s0, cfg)
torch.cuda.synchronize()
def loop(n=20):
    gc.collect(); gc.disable()
    evs = []
    for _ in range(n):
        flush.fill_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(); cs.run_deer(k, s0, cfg); b.record()
        evs.append((a, b))
    torch.cuda.synchronize(); gc.enable()
    return [round(a.elapsed_time(b), 3) for a, b in evs]
mode = sys.argv[1]
if mode == "sampler":
    with bench.ClockSampler(0) as clk:
        x = loop(); y = loop()
    print("sampler", x, "\n       ", y, clk.summary())
else:
    x = loop(); y = loop()
    print("plain  ", x, "\n       ", y)

"""Benchmark: converged samples/s of a 100K-step HMC chain solved in parallel
across its length (BASELINE.json configs[1]: HMC on the 2D Rosenbrock,
eps=0.5, L=8, T=100,000, diagonal quasi-Newton with clip=1 -- the only setting
the reference itself converges on).

A "step" is one complete run_deer solve of the chain (all Newton iterations to
convergence) from pre-drawn noise.  ``value`` times the solve with the noise
already resident in HBM; ``e2e`` goes through the public API from pinned host
noise (H2D of the noise tables, solve, D2H of the trace) every step.  L2 is
flushed (256 MiB write) between timed steps, outside the timed region.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "converged samples/s, 100K-step HMC chain solved in parallel (Newton iterations to convergence)"
T_DEFAULT = 100_000
EPS, LSTEPS = 0.5, 8
ROSEN = dict(a=0.0, b=0.1, scale1=1.0, scale2=1.0)


def workload(T):
    """The one workload description both arms print (same_config)."""
    return f"HMC Rosenbrock(b=0.1,s2=1) eps={EPS} L={LSTEPS} T={T}, diag quasi-Newton clip=1, s0=0"


def traffic(key):
    """DRAM bytes per launch of a kernel at a bench workload, from its committed
    ncu capture (profiles/r01_traffic.json); None when not captured."""
    try:
        with open(os.path.join(ROOT, "profiles", "r01_traffic.json")) as fh:
            return int(json.load(fh)[key]["bytes"])
    except Exception:
        return None


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


POLL_S = float(os.environ.get("CS_BENCH_POLL_MS", "5")) / 1e3


_POLLER = r"""
import json, sys, time
import pynvml
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(int(sys.argv[1]))
period = float(sys.argv[2])
mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
# the first queries of a process are slow (and hold the driver's lock): make
# them here, before the parent starts its timed region
for _ in range(3):
    pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
    pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
sys.stdout.write("ready\n"); sys.stdout.flush()
import select
samples, bits = [], 0
while not select.select([sys.stdin], [], [], period)[0]:
    try:
        samples.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
        bits |= pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
    except Exception:
        pass
sys.stdout.write(json.dumps({"samples": samples, "bits": bits, "max": mx}) + "\n"); sys.stdout.flush()
"""


class ClockSampler:
    """SM clocks and throttle reasons sampled (NVML, every POLL_S) during the timed
    region, by a child process: a poller thread in this process competes for the
    GIL with the solve's host path (measured: 0.43 -> 0.57 ms per headline step)."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "hw_power_brake_slowdown": 0x80, "sw_power_cap": 0x4}

    def __init__(self, gpu_index=0):
        self.gpu = gpu_index
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._p = None

    def __enter__(self):
        import subprocess

        try:
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[self.gpu]) if vis and vis.split(",")[self.gpu].strip().isdigit() else self.gpu
            self._p = subprocess.Popen([sys.executable, "-c", _POLLER, str(idx), str(POLL_S)], stdin=subprocess.PIPE,
                                       stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            if self._p.stdout.readline().strip() != "ready":
                self._p = None
        except Exception:
            self._p = None
        return self

    def __exit__(self, *a):
        if self._p is None:
            return
        try:
            out, _ = self._p.communicate("stop\n", timeout=30)
            r = json.loads(out.strip().splitlines()[-1])
            self.samples, self.max_mhz = r["samples"], r["max"]
            self.reasons = {n for n, b in self.REASONS.items() if r["bits"] & b}
        except Exception:
            self._p.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"]}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples), "sampler": "child process (NVML)"}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ---------------------------------------------------------------------------
# reference arm: the CPU oracle port on the host cores


def cpu_solve(T, seed=0):
    import oracle as O

    k = O.HmcKernel(O.rosenbrock(**ROSEN), EPS, LSTEPS, seed=seed, T=T)
    t0 = time.perf_counter()
    res = O.run_deer(k, np.zeros(2), O.DeerConfig(mode="diag-stochastic", clip=1.0))
    return time.perf_counter() - t0, res


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from oracle.scan import build_lib, workers_default

    build_lib()
    cores = workers_default()
    T = args.T
    for _ in range(args.warmup):
        cpu_solve(T)
    times, iters = [], []
    for _ in range(args.steps):
        dt, res = cpu_solve(T)
        times.append(dt)
        iters.append(res.iterations)
    tot = float(np.sum(times))
    value = args.steps * T / tot
    line = {"metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (counter-RNG noise)",
            "impl": "reference",
            "config": {"workload": workload(T), "T": T, "newton_iterations": int(np.median(iters))},
            "cpu_baseline": {"value": value, "unit": "samples/s", "cores": cores, "kind": "port",
                             "sample": f"full T={T} chain solve per step (oracle/: numpy f_t + pthread C scan)"},
            "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(line)
    return 0


# ---------------------------------------------------------------------------
# the B200 arm


def run_gpu(args):
    import torch
    import torch.distributed as dist

    import paper_2508_18413_b200 as cs
    from paper_2508_18413_b200 import _lib

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1 or not args.no_extras:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        dist.init_process_group("nccl", device_id=dev, rank=rank, world_size=world)
    dtype = torch.float32 if args.dtype == "f32" else torch.float64
    T = args.T
    seed = rank  # replicas: each rank solves its own chain (weak scaling)
    model = cs.model_logp_grad_hvp(cs.rosenbrock(**ROSEN))
    kern = cs.HmcKernel(model, EPS, LSTEPS, seed=seed, T=T, dtype=dtype)
    cfg = cs.DeerConfig(mode="diag-stochastic", clip=1.0)
    s0 = torch.zeros(2, dtype=dtype, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    # pinned host copies of the pre-drawn noise (the e2e inputs)
    mom_dev = kern.noise.table("momentum", dtype)
    logu_dev = kern.noise.table("u", torch.float64, log_uniform=True)
    mom_host = mom_dev.cpu().pin_memory()
    logu_host = logu_dev.cpu().pin_memory()
    trace_host = torch.empty((T, 2), dtype=dtype).pin_memory()
    h2d = mom_host.numel() * mom_host.element_size() + logu_host.numel() * logu_host.element_size()
    d2h = trace_host.numel() * trace_host.element_size()

    def solve():
        return cs.run_deer(kern, s0, cfg)

    res = None
    for _ in range(args.warmup):
        res = solve()
    if res is None:  # --warmup 0: one untimed solve still fixes the iteration count
        res = solve()
    torch.cuda.synchronize()
    iters = res.iterations

    kernel_ms = []

    def solve_rec():
        r = solve()
        kernel_ms.append(r.stats.get("device_ms", float("nan")))
        return r

    def timed(fn):
        # the collector stays off inside the timed region (a collection pause in
        # the host path would land in one step); objects are freed at the end
        gc.collect()
        gc.disable()
        # untimed pre-roll, results held at once: the timed loop keeps one step's
        # result alive while the next allocates, and the allocator must already
        # own blocks for both (otherwise step 2 pays a cudaMalloc: 2-100 ms)
        keep = []
        for _ in range(3):
            flush.fill_(1.0)
            keep.append(fn())
        torch.cuda.synchronize()
        del keep
        evs = []
        host = []
        for _ in range(args.steps):
            h0 = time.perf_counter()
            flush.fill_(1.0)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            h1 = time.perf_counter()
            a.record()
            out = fn()
            b.record()
            h2 = time.perf_counter()
            evs.append((a, b))
            host.append((round((h1 - h0) * 1e3, 3), round((h2 - h1) * 1e3, 3)))
        torch.cuda.synchronize()
        gc.enable()
        if os.environ.get("CS_BENCH_STEPS"):
            print("steps", [round(a.elapsed_time(b), 3) for a, b in evs], file=sys.stderr)
            print("host", host[:4], file=sys.stderr)
            print("kernel", [round(x, 3) for x in kernel_ms[-args.steps:]][:4], file=sys.stderr)
        return sum(a.elapsed_time(b) for a, b in evs), out

    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        ms_dev, res = timed(solve_rec)
        kernel_step_ms = float(np.mean(kernel_ms[-args.steps:]))

        def e2e_step():
            kern.noise.load("momentum", mom_host, dtype=dtype)
            kern.noise.load("u", logu_host, dtype=torch.float64, log_uniform=True)
            r = solve()
            trace_host.copy_(r.trace, non_blocking=True)
            return r

        ms_e2e, _ = timed(e2e_step)
    torch.cuda.synchronize()
    if world > 1:
        t = torch.tensor([ms_dev, ms_e2e], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_dev, ms_e2e = t.tolist()
        dist.barrier()

    value = world * args.steps * T / (ms_dev / 1e3)
    e2e_value = world * args.steps * T / (ms_e2e / 1e3)
    # dominant kernel: the persistent solver (one launch per solve); its
    # algorithmic bytes per Newton pass: read guess rows + noise rows, write the
    # next guess (+ int32 fail stamps), i.e. T*(2 D s + D s + 8) + T*D*s
    es = 4 if dtype == torch.float32 else 8
    passes = iters + 1 if res.stats.get("stop_reason") != _lib.CS_STOP_NOFAIL else iters
    bytes_per_launch = T * (2 * es + 2 * es + 8) * passes + T * 2 * es * iters + T * 4
    per_launch_s = ms_dev / 1e3 / args.steps
    hbm, src = peaks()
    achieved = bytes_per_launch / per_launch_s / 1e9
    roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
            "traffic": traffic(f"deer_persistent_hmc_rosen_T{T}") if dtype == torch.float32 else None,
            "kernel": "cs::deer_persistent<Hmc<2,f,Rosenbrock>,DIAG> (whole solve)",
            "peak_source": src, "algorithmic_bytes_per_launch": bytes_per_launch,
            "note": "whole-solve working set (3.6 MB) is L2-resident: the kernel is bound by the grid "
                    "barrier and dependent f64 leapfrog chains, not HBM (profiles/r02_ncu_hmc_fused_solver.md); "
                    "the HBM-bound scan is scan_roofline"}

    # f64 companion (the reference computes in f64): the same solve, device-resident
    f64 = f64_companion(cs, dev, T, args) if not args.no_extras and dtype == torch.float32 else None

    # the T-sharded driver on BASELINE cfg 5
    shard = t_sharded_gibbs(cs, dev, world, rank) if not args.no_extras else None
    scan_roof = None
    cpu_base = None
    if rank == 0 and not args.no_extras:
        scan_roof = scan_roofline(cs, dev, hbm, src)
        cpu_base = cpu_baseline_sample(args)
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_dev / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": args.dtype,
                "data": "synthetic (counter-RNG noise, reference seed 0 per rank)",
                "config": {"workload": workload(T),
                           "T": T, "newton_iterations": iters, "parallelism": f"replicas x{world}",
                           "l2": "flushed (256 MiB write) between timed steps",
                           "solver": res.stats},
                "e2e": {"value": e2e_value, "unit": "samples/s", "h2d_bytes_per_step": h2d,
                        "d2h_bytes_per_step": d2h, "ms_per_step": ms_e2e / args.steps,
                        "gpu_launches": args.steps * int(res.stats.get("launches", 3))},
                "gpu_launches": args.steps * int(res.stats.get("launches", 3)),
                "kernel_ms_per_step": kernel_step_ms,
                "roofline": roof, "scan_roofline": scan_roof, "cpu_baseline": cpu_base,
                **({"t_sharded": shard} if shard is not None else {}),
                **({"f64": f64} if f64 is not None else {}),
                "clocks": clk.summary()}
        emit(line)
    if dist.is_initialized():
        dist.destroy_process_group()
    return 0


def f64_companion(cs, dev, T, args):
    """The headline solve with states and elements in f64 (the reference's
    dtype): device-resident timing like ``value``; reported beside it."""
    import torch

    try:
        k = cs.HmcKernel(cs.model_logp_grad_hvp(cs.rosenbrock(**ROSEN)), EPS, LSTEPS, seed=0, T=T,
                         dtype=torch.float64)
        cfg = cs.DeerConfig(mode="diag-stochastic", clip=1.0)
        s0 = torch.zeros(2, dtype=torch.float64, device=dev)
        for _ in range(max(3, args.warmup)):
            r = cs.run_deer(k, s0, cfg)
        n = max(5, min(args.steps, 20))
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ker = []
        a.record()
        for _ in range(n):
            r = cs.run_deer(k, s0, cfg)
            ker.append(r.stats.get("device_ms", float("nan")))
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / n
        return {"value": T / (ms / 1e3), "unit": "samples/s", "ms_per_step": ms, "kernel_ms_per_step": float(np.mean(ker)),
                "newton_iterations": r.iterations, "steps": n, "dtype": "f64", "solver": r.stats}
    except Exception as e:  # reported, never required
        return {"error": f"{type(e).__name__}: {e}"[:300]}


def t_sharded_gibbs(cs, dev, world, rank, reps=3):
    """BASELINE cfg 5 (Gibbs eight schools, T = 1M, diag x3 + preconditioner)
    solved with T sharded over the ranks: contiguous shards, three small NCCL
    all-gathers per Newton iteration (sharded.py).  Device time per solve, max
    over ranks; reported next to the headline, never instead of it."""
    import torch
    import torch.distributed as dist

    try:
        from paper_2508_18413_b200.sharded import run_deer_sharded

        T = 1_000_000
        k = cs.GibbsKernel(cs.generate_eight_schools(), seed=0, T=T, dtype=torch.float32)
        cfg = cs.DeerConfig(mode="diag-stochastic", hutchinson_samples=3,
                            preconditioner=k.recommended_preconditioner(), max_iters=400)
        s0 = k.initial_state()
        r = run_deer_sharded(k, s0, cfg)  # warm-up
        ms = []
        for _ in range(reps):
            dist.barrier()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            r = run_deer_sharded(k, s0, cfg)
            b.record()
            torch.cuda.synchronize()
            ms.append(a.elapsed_time(b))
        t = torch.tensor([float(np.median(ms))], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        m = float(t.item())
        return {"workload": "cfg5 Gibbs eight schools T=1M, diag-stochastic x3 + preconditioner, fp32",
                "world": world, "ms_per_solve": m, "samples_per_s": T / (m / 1e3), "iterations": r.iterations,
                "converged": bool(r.converged), "rows_on_rank0": [int(r.lo), int(r.hi)] if rank == 0 else None,
                "collectives_per_iteration": 3, "timing": f"median of {reps} solves, max over ranks"}
    except Exception as e:  # reported, never required for the headline line
        return {"error": f"{type(e).__name__}: {e}"[:300]}


def scan_roofline(cs, dev, hbm, src):
    """The standalone diagonal scan at an HBM-sized problem (north_star: the
    diag/block scans are HBM-bound; 12 B per element in fp32)."""
    import torch

    T, D = 1 << 24, 18  # SURVEY.md 8d's large synthetic (3.6 GB of j, u, s): well past L2
    g = torch.Generator(device=dev).manual_seed(0)
    j = (torch.rand((T, D), generator=g, device=dev) * 1.8 - 0.9).float()
    u = torch.randn((T, D), generator=g, device=dev).float()
    s0 = torch.zeros(D, device=dev)
    out = torch.empty_like(u)
    el = cs.DiagElements(j, u)
    for _ in range(3):
        cs.parallel_affine_solve(el, s0, out=out)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    times = []
    for _ in range(10):
        flush.fill_(0.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        cs.parallel_affine_solve(el, s0, out=out)
        b.record()
        torch.cuda.synchronize()
        times.append(a.elapsed_time(b))
    ms = float(np.median(times))
    byts = 12 * T * D
    ach = byts / (ms / 1e3) / 1e9
    return {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
            "traffic": traffic(f"scan_local_diag_f32_T{T}_D{D}"),
            "kernel": "cs::scan_local<float> + scan_local_carry + scan_local_fixup (one scan)", "T": T, "D": D,
            "ms": ms, "peak_source": src, "algorithmic_bytes": byts,
            "note": "local scan per CTA range (j, u read once, s written once) + f64-exact fix-up of each "
                    "range's leading tiles while prod a != 0; profiles/r02_ncu_scan_local_T16M_D18.md"}


def cpu_baseline_sample(args):
    try:
        from oracle.scan import build_lib, workers_default

        build_lib()
        dt, res = cpu_solve(args.T)
        return {"value": args.T / dt, "unit": "samples/s", "cores": workers_default(), "kind": "port",
                "sample": f"one full T={args.T} solve ({res.iterations} Newton iterations), oracle/ numpy+C"}
    except Exception as e:  # the CPU baseline is reported, never required
        return {"value": None, "unit": "samples/s", "cores": os.cpu_count(), "kind": "port",
                "sample": f"unavailable: {e}"}


_JSON_OUT = None


def emit(line):
    """The ONE JSON line, on the real stdout (libraries' chatter -- e.g. NCCL's
    version banner at communicator init -- is routed to stderr by main())."""
    out = _JSON_OUT or sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


def main():
    global _JSON_OUT
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)  # anything else written to fd 1 (C or Python) lands on stderr
    sys.stdout = sys.stderr
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--dtype", default="f32", choices=["f32", "f64"])
    ap.add_argument("--T", type=int, default=T_DEFAULT)
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--sharded", action="store_true", help="(kept for compatibility: t_sharded always runs)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())

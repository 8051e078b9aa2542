import ctypes, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_18413_b200 as cs
from paper_2508_18413_b200 import _lib
from paper_2508_18413_b200.samplers import hmc_chain_system
m = cs.model_logp_grad_hvp(cs.rosenbrock())
k = hmc_chain_system(m, eps=0.2, L=16, seed=5, T=48, leapfrog_mode="parallel",
                     leapfrog_cfg=cs.DeerConfig(mode="block2x2-stochastic", engine="host"))
x0 = np.array([0.5, -0.5])
tr = cs.sequential_evaluate(k, x0)
S = torch.cat([torch.as_tensor(x0, device="cuda")[None], tr[:-1]])
ts = torch.arange(1, 49, device="cuda")
# reproduce the proposal inputs
xi = k.noise.table("momentum", torch.float64)[ts]
mass = torch.ones(2, dtype=torch.float64, device="cuda")
v_half = torch.sqrt(mass) * xi + 0.5 * 0.2 * m.grad(S)
system = k.leapfrog_system()
s0s = torch.cat([S, v_half], dim=1).contiguous()
B = 48
finals = torch.empty_like(s0s); info = torch.empty((B, 4), dtype=torch.int32, device="cuda"); err = torch.empty(B, dtype=torch.int64, device="cuda")
c = _lib.cs_deer_config(); c.mode = _lib.CS_MODE_BLOCK; c.atol, c.rtol = 1e-4, 1e-3; c.max_iters = 51; c.hutchinson_samples = 1; c.damping = 1.0; c.clip = float("inf"); c.preconditioner = 0
d = system.desc()
lib = _lib.load()
_lib.check(lib.cs_leapfrog_batch_solve(ctypes.byref(d), ctypes.byref(c), _lib.CS_F64, B, _lib.ptr(s0s), _lib.ptr(finals), _lib.ptr(info), _lib.ptr(err), _lib.stream_ptr()))
ih = info.cpu().numpy()
for b in range(B):
    try:
        r = cs.run_deer(system, s0s[b], cs.DeerConfig(mode="block2x2-stochastic", engine="host"))
        ref = (int(r.converged), r.iterations, r.delta_history[:4].round(6).tolist(), r.delta_history[-3:].round(6).tolist())
    except cs.ChainDivergedError as e:
        ref = ("raise", str(e)[:60])
    if ih[b][0] != 1 or (ref[0] != 1):
        print(b, "batched", ih[b].tolist(), int(err[b]), "| host", ref)

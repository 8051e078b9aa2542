import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_2508_18413_b200 as cs
dev = "cuda"
def seq(J, u, s0):
    s = s0.copy(); out = []
    for t in range(len(J)):
        s = J[t] @ s + u[t]; out.append(s)
    return np.array(out)
for D, T, kind in [(16, 16, "eye"), (16, 16, "diag"), (16, 16, "rand"), (16, 2000, "rand"), (100, 2049, "rand"), (64, 64, "rand")]:
    rng = np.random.default_rng(1)
    if kind == "eye": J = np.repeat(np.eye(D)[None], T, 0)
    elif kind == "diag": J = np.stack([np.diag(rng.uniform(0.5, 1.0, D)) for _ in range(T)])
    else: J = rng.normal(size=(T, D, D)) * (0.9 / (2 * np.sqrt(D)))
    u = rng.normal(size=(T, D)); s0 = rng.normal(size=D)
    tt = lambda x: torch.as_tensor(x, dtype=torch.float32, device=dev)
    Jd, ud, s0d = (tt(x).double().cpu().numpy() for x in (J, u, s0))
    want = seq(Jd, ud, s0d)
    got = cs.parallel_affine_solve(cs.DenseElements(tt(J), tt(u)), tt(s0)).double().cpu().numpy()
    err = np.abs(got - want).max(axis=1)
    bad = np.nonzero(err > 1e-3)[0]
    print(os.environ.get("CS_DENSE_TREE"), D, T, kind, "maxerr", err.max(), "first bad", bad[:5], flush=True)

"""Time the dense scan at cfg 3's shape (T, D = 100, f32) through parallel_affine_solve."""
import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_18413_b200 as cs
T = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
D = 100
g = torch.Generator(device="cuda").manual_seed(0)
J = torch.randn((T, D, D), generator=g, device="cuda") * (0.45 / np.sqrt(D))
u = torch.randn((T, D), generator=g, device="cuda")
s0 = torch.randn(D, generator=g, device="cuda")
for _ in range(2):
    cs.parallel_affine_solve(cs.DenseElements(J, u), s0)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(5):
    cs.parallel_affine_solve(cs.DenseElements(J, u), s0)
b.record()
torch.cuda.synchronize()
print(f"dense scan T={T} D={D} f32: {a.elapsed_time(b) / 5:.3f} ms  (CS_TREE_DBG={os.environ.get('CS_TREE_DBG')}, CS_DENSE_TREE={os.environ.get('CS_DENSE_TREE')})", flush=True)

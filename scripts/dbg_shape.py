import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_1511_03296_b200 as fbs
H, W = int(sys.argv[1]), int(sys.argv[2])
rng = np.random.default_rng(H * 100 + W)
rgb = rng.integers(0, 256, (1, H, W, 3), dtype=np.uint8)
t = rng.uniform(0, 1, (1, 1, H, W)).astype(np.float32)
c = rng.uniform(0.1, 1, (1, H, W)).astype(np.float32)
g = fbs.grid_build(torch.from_numpy(rgb).cuda(), 8.0, 4.0, 3.0)
torch.cuda.synchronize(); print('built', flush=True)
print(g.M, g.levels, g.info(), flush=True)
x = fbs.solve(g, torch.from_numpy(t).cuda(), torch.from_numpy(c).cuda(), 10.0, precond="hier", init="hier", mode="tol", tol=1e-6)
torch.cuda.synchronize(); print('solved', flush=True)

"""Two C2 solves through the graph loop (for ncu launch lists of the loop kernels)."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2311_04362_b200 as itsk
p = itsk.gen_randsvd(200000, 200, 1e10, 1e-12, 0)
at = torch.from_numpy(p.a).cuda(); bt = torch.from_numpy(p.b).cuda()
cfg = itsk.SolverConfig(d=4000)
for _ in range(2):
    r = itsk.iterative_sketching(at, bt, cfg, residuals="last")
torch.cuda.synchronize()
print("iters", r.iterations)

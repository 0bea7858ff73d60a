"""Solve with the step-wise loop (no graph) so ncu sees each loop kernel."""
import sys, os
sys.path.insert(0, os.getcwd())
import torch
import paper_2311_04362_b200 as itsk
from bench import CONFIGS
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
m, n, kappa, beta, d, zeta = CONFIGS[name]
p = itsk.gen_randsvd(m, n, kappa, beta, 0)
at = torch.from_numpy(p.a).cuda(); bt = torch.from_numpy(p.b).cuda()
cfg = itsk.SolverConfig(d=d, zeta=zeta, max_iters=4)
r = itsk.iterative_sketching(at, bt, cfg, residuals="last", use_graph=False)
torch.cuda.synchronize()
r = itsk.iterative_sketching(at, bt, cfg, residuals="last", use_graph=False)
torch.cuda.synchronize()

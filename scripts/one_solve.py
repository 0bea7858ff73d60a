"""One warm solve + one measured solve of a bench config (for ncu launch lists)."""
import sys, os
sys.path.insert(0, os.getcwd())
import torch
import paper_2311_04362_b200 as itsk
from bench import CONFIGS
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
variant = sys.argv[2] if len(sys.argv) > 2 else "basic"
m, n, kappa, beta, d, zeta = CONFIGS[name]
p = itsk.gen_randsvd(m, n, kappa, beta, 0)
at = torch.from_numpy(p.a).cuda(); bt = torch.from_numpy(p.b).cuda()
cfg = itsk.SolverConfig(d=d, zeta=zeta, variant=variant)
r = itsk.iterative_sketching(at, bt, cfg, residuals="last")
torch.cuda.synchronize()
print("MEASURED-SOLVE-START", flush=True)
r = itsk.iterative_sketching(at, bt, cfg, residuals="last")
torch.cuda.synchronize()
print("iters", r.iterations, r.trace.stop_reason)

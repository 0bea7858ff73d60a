"""cProfile of the host side of repeated solves (where does Python spend the
time the GPU does not cover?):  python scripts/host_profile.py [c1|c2] [reps]"""
import cProfile, os, pstats, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2311_04362_b200 as itsk
from bench import CONFIGS, make_problem

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
m, n, kappa, beta, d, zeta = CONFIGS[name]
p, _, _ = make_problem(name, 0)
dev = torch.device("cuda")
at = p.a if isinstance(p.a, torch.Tensor) else torch.from_numpy(p.a).to(dev)
bt = p.b if isinstance(p.b, torch.Tensor) else torch.from_numpy(p.b).to(dev)
cfg = itsk.SolverConfig(d=d, zeta=zeta)
for _ in range(5):
    itsk.iterative_sketching(at, bt, cfg, residuals="all")
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(reps):
    itsk.iterative_sketching(at, bt, cfg, residuals="all")
pr.disable()
torch.cuda.synchronize()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(22)

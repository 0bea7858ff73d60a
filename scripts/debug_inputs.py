import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2311_04362_b200 as itsk
p = itsk.gen_randsvd(3000, 40, 1e8, 1e-6, 2)
cfg = itsk.SolverConfig(d=800, variant="momentum", rng_seed=2)
def show(tag, r):
    print(tag, r.iterations, r.trace.stop_reason, r.trace.normest, r.trace.condest, r.solution[:3], r.trace.iterates[0][:3])
r1 = itsk.iterative_sketching(p.a, p.b, cfg); show("host1", r1)
r1b = itsk.iterative_sketching(p.a, p.b, cfg); show("host2", r1b)
at = torch.from_numpy(p.a).cuda(); bt = torch.from_numpy(p.b).cuda()
r2 = itsk.iterative_sketching(at, bt, cfg); show("dev", r2)
r2b = itsk.iterative_sketching(at, bt, cfg, use_graph=False); show("dev-steps", r2b)
big = torch.zeros((3000, 48), dtype=torch.float64, device="cuda"); big[:, :40] = at
r3 = itsk.iterative_sketching(big[:, :40], bt, cfg); show("view", r3)
for a, b in [(r1, r1b), (r1, r2), (r2, r2b), (r1, r3)]:
    print(np.array_equal(a.solution, b.solution), np.array_equal(a.trace.iterates[0], b.trace.iterates[0]), a.trace.normest == b.trace.normest)

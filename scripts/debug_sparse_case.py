import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2311_04362_b200 as itsk
from oracle import itsketch_oracle as orc
m, n, d, seed = 465, 80, 1383, 2
p = itsk.gen_sparse(m, n, seed)
a, b = p.a.tocsr(), p.b
x_o, t_o = orc.iterative_sketching(a, b, orc.Config(d=d, variant="momentum", rng_seed=seed))
r_d = itsk.iterative_sketching(a, b, itsk.SolverConfig(d=d, variant="momentum", rng_seed=seed), residuals="all")
U = 2.0**-53
def deltas(iterates):
    rs = [b - a @ x for x in iterates]
    return [float(np.linalg.norm(rs[i+1] - rs[i])) for i in range(len(rs)-1)], [float(np.linalg.norm(r)) for r in rs]
do, ro = deltas(t_o.iterates)
dd, rd = deltas(r_d.trace.iterates)
print("normest/condest oracle", t_o.normest, t_o.condest, "device", r_d.trace.normest, r_d.trace.condest)
thr_o = U * (t_o.normest * np.linalg.norm(t_o.iterates[-1]) + 0.04 * t_o.condest * ro[-1])
print("threshold ~", thr_o, "||r||", ro[-1], rd[-1], "stop", t_o.stop_reason, len(do), r_d.trace.stop_reason, len(dd))
for i in range(max(len(do), len(dd))):
    print(i, f"{do[i]:.3e}" if i < len(do) else "-", f"{dd[i]:.3e}" if i < len(dd) else "-")

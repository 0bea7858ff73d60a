"""A/B of one env setting on full solves in one process (same box, same
instance, alternating): python scripts/solve_ab.py CONFIG VARIANT ENV=A ENV=B [reps]
e.g. python scripts/solve_ab.py c4 momentum ITSK_SKETCH_SWEEP=-1 ITSK_SKETCH_SWEEP=0 5"""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2311_04362_b200 as itsk
from bench import CONFIGS, make_problem

cfgname, variant, ea, eb = sys.argv[1:5]
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 5
m, n, kappa, beta, d, zeta = CONFIGS[cfgname]
p, _, _ = make_problem(cfgname, 0)
dev = torch.device("cuda")
at = p.a if isinstance(p.a, torch.Tensor) else torch.from_numpy(p.a).to(dev)
bt = p.b if isinstance(p.b, torch.Tensor) else torch.from_numpy(p.b).to(dev)
cfg = itsk.SolverConfig(d=d, zeta=zeta, variant=variant)


def setenv(kv):
    k, v = kv.split("=", 1)
    if v == "":
        os.environ.pop(k, None)
    else:
        os.environ[k] = v


times = {ea: [], eb: []}
for r in range(reps + 1):
    for kv in (ea, eb):
        setenv(kv)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        res = itsk.iterative_sketching(at, bt, cfg, residuals="last")
        e1.record()
        torch.cuda.synchronize()
        if r > 0:
            times[kv].append(e0.elapsed_time(e1))
for kv, ts in times.items():
    print(f"{cfgname} {variant} {kv}: median {statistics.median(ts):.2f} ms  min {min(ts):.2f}  all "
          + " ".join(f"{t:.1f}" for t in ts), flush=True)

"""Host enqueue time of one C2 solve vs its device time: if the host needs
about as long to enqueue the solve as the GPU needs to run it, launch
overhead is on the critical path."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
import paper_2311_04362_b200 as itsk
from bench import CONFIGS, make_problem

m, n, kappa, beta, d, zeta = CONFIGS["c2"]
p, _, _ = make_problem("c2", 0)
dev = torch.device("cuda")
at = torch.from_numpy(p.a).to(dev); bt = torch.from_numpy(p.b).to(dev)
cfg = itsk.SolverConfig(d=d, zeta=zeta)
orig = torch.cuda.Stream.synchronize
marks = {}


def sync(self):
    marks.setdefault("enq", time.perf_counter())
    return orig(self)


for rep in range(6):
    torch.cuda.synchronize()
    marks.clear()
    torch.cuda.Stream.synchronize = sync
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    t0 = time.perf_counter()
    e0.record()
    res = itsk.iterative_sketching(at, bt, cfg, residuals="all")
    e1.record()
    torch.cuda.Stream.synchronize = orig
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    if rep >= 2:
        print(f"host enqueue {1e3 * (marks['enq'] - t0):.3f} ms  device {e0.elapsed_time(e1):.3f} ms  "
              f"wall {1e3 * (t1 - t0):.3f} ms")

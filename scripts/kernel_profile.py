"""Warm per-kernel device time of one solve via torch.profiler (CUPTI; no
cache flush between kernels, unlike ncu's launch list).
Usage: python scripts/kernel_profile.py [c2|c3] [variant]"""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
from torch.profiler import ProfilerActivity, profile

import paper_2311_04362_b200 as itsk
from bench import CONFIGS, make_problem

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
variant = sys.argv[2] if len(sys.argv) > 2 else "basic"
m, n, kappa, beta, d, zeta = CONFIGS[name]
p, _, _ = make_problem(name, 0)
dev = torch.device("cuda")
at = p.a if isinstance(p.a, torch.Tensor) else torch.from_numpy(p.a).to(dev)
bt = p.b if isinstance(p.b, torch.Tensor) else torch.from_numpy(p.b).to(dev)
cfg = itsk.SolverConfig(d=d, zeta=zeta, variant=variant)
for _ in range(3):
    itsk.iterative_sketching(at, bt, cfg, residuals="all")
torch.cuda.synchronize()
reps = 5
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(reps):
        itsk.iterative_sketching(at, bt, cfg, residuals="all")
    torch.cuda.synchronize()
agg = {}
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA and e.device_time_total > 0:
        k = e.name.replace("(anonymous namespace)::", "").replace("itsk::", "").split("(")[0][:60]
        c, t = agg.get(k, (0, 0.0))
        agg[k] = (c + 1, t + e.device_time_total)
tot = sum(t for _, t in agg.values())
print(f"{name} {variant}: per solve, warm (torch.profiler / CUPTI), {reps} solves")
print(f"{'kernel':60s} {'per solve':>9s} {'us/solve':>9s} {'us each':>8s} {'share':>6s}")
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:60s} {c / reps:9.1f} {t / reps:9.1f} {t / c:8.2f} {100 * t / tot:5.1f}%")
print(f"{'total kernel time per solve':60s} {'':9s} {tot / reps:9.1f}")

"""Probe of the solver's size limits in n (the triangular / estimate kernels are single-CTA or one-cluster kernels):
    python scripts/size_limits.py"""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2311_04362_b200 as itsk

for n, d, m in ((2500, 10000, 30000), (3000, 12000, 30000), (4096, 16384, 40000), (5000, 15000, 40000),
                (6000, 18000, 40000), (6500, 19500, 40000), (9000, 27000, 50000)):
    g = torch.Generator(device="cuda").manual_seed(n)
    a = torch.randn(m, n, dtype=torch.float64, device="cuda", generator=g)
    x = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
    b = a @ x + 1e-6 * torch.randn(m, dtype=torch.float64, device="cuda", generator=g)
    try:
        t0 = time.perf_counter()
        res = itsk.iterative_sketching(a, b, itsk.SolverConfig(d=d, variant="momentum"))
        torch.cuda.synchronize()
        err = float(np.linalg.norm(res.solution - x.cpu().numpy()) / np.linalg.norm(x.cpu().numpy()))
        print(f"n={n} d={d} m={m}: {res.trace.stop_reason} in {res.iterations} it., {1e3 * (time.perf_counter() - t0):.0f} ms, "
              f"|x - x*|/|x*| = {err:.2e}", flush=True)
    except Exception as e:  # noqa: BLE001
        print(f"n={n} d={d} m={m}: {type(e).__name__}: {str(e)[:140]}", flush=True)
    del a, b
    torch.cuda.empty_cache()

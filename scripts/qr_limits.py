import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2311_04362_b200 as itsk
for d, n in ((30000, 100), (30000, 2000), (50000, 500), (50000, 2000), (100000, 200), (100000, 2000), (200000, 1000), (400000, 50)):
    a = torch.randn(d, n, dtype=torch.float64, device="cuda")
    try:
        t0 = time.perf_counter()
        f = itsk.householder_qr_econ(a)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        r = f.r
        # check R'R = A'A
        g = a.T @ a
        err = float(torch.linalg.matrix_norm(r.T @ r - g) / torch.linalg.matrix_norm(g))
        print(f"d={d} n={n}: ok {1e3*dt:.1f} ms, |R'R - A'A|/|A'A| = {err:.1e}", flush=True)
    except Exception as e:
        print(f"d={d} n={n}: {type(e).__name__}: {str(e)[:120]}", flush=True)
    del a
    torch.cuda.empty_cache()

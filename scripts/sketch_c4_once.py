"""One S·[A|b] at the C4 shape on a random A (for ncu / timing):
    python scripts/sketch_c4_once.py [m n d zeta reps]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2311_04362_b200 as itsk
m, n, d, zeta = (int(v) for v in sys.argv[1:5]) if len(sys.argv) > 4 else (4000000, 2000, 24000, 8)
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 3
g = torch.Generator(device="cuda").manual_seed(0)
A = torch.randn(m, n, dtype=torch.float64, device="cuda", generator=g)
b = torch.randn(m, dtype=torch.float64, device="cuda", generator=g)
s = itsk.sparse_sign_new(d, m, zeta, 0)
for r in range(reps):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    w = s.apply_dense(A, b)
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(f"sketch m={m} n={n} d={d} zeta={zeta}: {dt * 1e3:.2f} ms  ({8 * m * (n + 1) / dt / 1e9:.0f} GB/s algorithmic, "
          f"{zeta * 8 * m * (n + 1) / dt / 1e9:.0f} GB/s gathered)", flush=True)

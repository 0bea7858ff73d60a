"""Time the sparse pass kernels (for ncu launch lists): gen_sparse(m, n), 5 passes."""
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2311_04362_b200 as itsk
m, n = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
p = itsk.gen_sparse(m, n, 0)
dev = torch.device("cuda", 0)
A = itsk.CsrMatrix.from_scipy(p.a, dev)
b = torch.from_numpy(p.b).to(dev)
x = torch.randn(n, dtype=torch.float64, device=dev)
r_out = torch.empty(m, dtype=torch.float64, device=dev)
r_prev = torch.zeros(m, dtype=torch.float64, device=dev)
for _ in range(3):
    A.pass_(b, x, r_out=r_out, r_prev=r_prev)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    A.pass_(b, x, r_out=r_out, r_prev=r_prev)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
alg = 24.0 * p.a.nnz + 8.0 * (m + 1) + 24.0 * m
print(f"sparse pass m={m} n={n}: {ms*1e3:.1f} us  {alg/ms/1e6:.0f} GB/s")

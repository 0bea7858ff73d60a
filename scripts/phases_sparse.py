"""Phase times of the sparse solve (CUDA events): plan, pattern, S·[A|b], QR, loop."""
import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2311_04362_b200 as itsk
from paper_2311_04362_b200 import linalg
m, n = int(sys.argv[1]), int(sys.argv[2])
d = 30 * n
p = itsk.gen_sparse(m, n, 0)
dev = torch.device("cuda", 0)
def ev():
    e = torch.cuda.Event(enable_timing=True); e.record(); return e
for rep in range(3):
    torch.cuda.synchronize()
    e0 = ev(); A = itsk.CsrMatrix.from_scipy(p.a, dev); e1 = ev()
    b = torch.from_numpy(p.b).to(dev)
    e2 = ev(); s = itsk.sparse_sign_new(d, m, 8, 0); e3 = ev()
    w = A.sketch(s, b); e4 = ev()
    r, z = linalg.qr_aug(w, n); e5 = ev()
    res = itsk.iterative_sketching(A, b, itsk.SolverConfig(d=d, max_iters=20), residuals="last"); e6 = ev()
    torch.cuda.synchronize()
    print(f"m={m} n={n} d={d}: plan {e0.elapsed_time(e1):.2f} pattern {e2.elapsed_time(e3):.2f} "
          f"sketch {e3.elapsed_time(e4):.2f} qr {e4.elapsed_time(e5):.2f} full solve {e5.elapsed_time(e6):.2f} ms")

"""S·[A|b] one-shot vs in row windows sized to stay L2-resident (itsk_sketch_rows)."""
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2311_04362_b200 as itsk
from paper_2311_04362_b200 import _lib
from paper_2311_04362_b200 import device as dv
m, n, d = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
dev = torch.device("cuda", 0)
A = torch.randn(m, n, dtype=torch.float64, device=dev)
b = torch.randn(m, dtype=torch.float64, device=dev)
s = itsk.sparse_sign_new(d, m, 8, 0)
lib = dv.lib(dev)
W = torch.empty(d, n + 1, dtype=torch.float64, device=dev)
ref = s.apply_dense(A, b)
def run(rows):
    if rows >= m:
        _lib.check(lib.itsk_sketch(dv.ptr(A), m, n, n, dv.ptr(b), dv.ptr(s.ptr_dev), dv.ptr(s.src_dev), d, 8, dv.ptr(W), n + 1, dv.stream_ptr()))
        return
    for k, r0 in enumerate(range(0, m, rows)):
        _lib.check(lib.itsk_sketch_rows(dv.ptr(A), m, n, n, dv.ptr(b), dv.ptr(s.ptr_dev), dv.ptr(s.src_dev), d, 8, dv.ptr(W), n + 1, r0, min(m, r0 + rows), 1 if k else 0, dv.stream_ptr()))
for mb in [0, 16, 32, 48, 64, 96]:
    rows = m if mb == 0 else max(1, (mb << 20) // (8 * n))
    run(rows); torch.cuda.synchronize()
    assert torch.equal(W, ref)
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(3): run(rows)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(f"m={m} n={n} d={d} window={'all' if mb == 0 else str(mb) + 'MB'}: {ms:.3f} ms  {8*m*(n+1)/ms/1e6:.0f} GB/s")

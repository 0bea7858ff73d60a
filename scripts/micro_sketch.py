"""Sketch S·[A|b] timing (C5 sweep point or a config shape).

    python scripts/micro_sketch.py m n d zeta [reps]
Prints device ms of the pattern generation and of the sketch kernel and the
sketch's algorithmic GB/s (8 m (n+1) bytes of [A|b] read once)."""
import ctypes, os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2311_04362_b200 import _lib
from paper_2311_04362_b200 import device as dv
from paper_2311_04362_b200.embed import pcg_state

m, n, d, zeta = (int(v) for v in sys.argv[1:5])
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 5
lib = _lib.lib_for_device(0)
dev = torch.device("cuda")
A = torch.randn(m, n, dtype=torch.float64, device=dev)
b = torch.randn(m, dtype=torch.float64, device=dev)
nnz = m * zeta
rows = torch.empty(nnz, dtype=torch.int32, device=dev)
neg = torch.empty(nnz, dtype=torch.uint8, device=dev)
sk_ptr = torch.empty(d + 1, dtype=torch.int32, device=dev)
sk_src = torch.empty(nnz, dtype=torch.int32, device=dev)
nb = ctypes.c_int64()
_lib.check(lib.itsk_pattern_workspace(d, m, zeta, ctypes.byref(nb)))
ws = dv.workspace(nb.value, dev)
W = torch.empty(d, n + 1, dtype=torch.float64, device=dev)
s = int(torch.cuda.current_stream().cuda_stream)
words, h, pend = pcg_state(0)


def pattern():
    _lib.check(lib.itsk_sparse_sign_pattern(d, m, zeta, words, h, pend, dv.ptr(rows), dv.ptr(neg), dv.ptr(sk_ptr),
                                            dv.ptr(sk_src), dv.ptr(ws), ws.numel(), s))


def sketch():
    _lib.check(lib.itsk_sketch(dv.ptr(A), m, n, n, dv.ptr(b), dv.ptr(sk_ptr), dv.ptr(sk_src), d, zeta, dv.ptr(W),
                               n + 1, s))


def timed(fn):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


tp = timed(pattern)
ts = timed(sketch)
print(f"sketch m={m} n={n} d={d} zeta={zeta}: pattern {tp:.3f} ms  sketch {ts:.3f} ms  "
      f"{8 * m * (n + 1) / ts / 1e6:.0f} GB/s (A read once)  {8 * zeta * m * (n + 1) / ts / 1e6:.0f} GB/s (zeta x A)")

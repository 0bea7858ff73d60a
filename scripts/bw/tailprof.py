"""Phase cycles of the loop tail kernel (thread 0), lib built with -DITSK_TAIL_PROBE:
  cd paper_2311_04362_b200/csrc && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \\
    -Xcompiler -fPIC --expt-relaxed-constexpr -I. -I../../include -DITSK_TAIL_PROBE -shared \\
    -o ../../scripts/bw/libtailprof.so capi.cu qr.cu qr2.cu qr_tsqr.cu trsv.cu pass.cu loop.cu pattern.cu sketch.cu \\
    -lcudart_static -lrt -ldl -lpthread"""
import ctypes, os, sys
sys.path.insert(0, os.getcwd())
from paper_2311_04362_b200 import _lib
lib = _lib.load(os.path.abspath("scripts/bw/libtailprof.so"))
lib.itsk_tail_profile_read.argtypes = [ctypes.c_void_p]
import torch
import paper_2311_04362_b200 as itsk
p = itsk.gen_randsvd(200000, 200, 1e10, 1e-12, 0)
at = torch.from_numpy(p.a).cuda(); bt = torch.from_numpy(p.b).cuda()
cfg = itsk.SolverConfig(d=4000)
out = (ctypes.c_ulonglong * 16)()
for _ in range(2):
    itsk.iterative_sketching(at, bt, cfg, residuals="last"); torch.cuda.synchronize()
lib.itsk_tail_profile_read(out)
r = itsk.iterative_sketching(at, bt, cfg, residuals="last"); torch.cuda.synchronize()
lib.itsk_tail_profile_read(out)
calls = out[15]
names = ["ctl copy", "(unused)", "control", "stage R+v", "trsv_t", "trsv_n", "update"]
print("tail calls", calls, "iterations", r.iterations)
for i, nm in enumerate(names):
    print(f"{nm:10s} {out[i] / max(calls, 1):9.0f} cycles/call")

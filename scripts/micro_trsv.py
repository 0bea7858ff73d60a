import sys, os, ctypes
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2311_04362_b200 import _lib
from paper_2311_04362_b200 import device as dv
n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
lib = _lib.lib_for_device(0)
rng = np.random.default_rng(0)
R = torch.from_numpy(np.triu(rng.standard_normal((n, n))) + (n + 2.0) * np.eye(n)).cuda()
c = torch.randn(n, dtype=torch.float64, device="cuda")
y = torch.empty_like(c)
s = dv.stream_ptr()
for _ in range(3):
    _lib.check(lib.itsk_trsv_pair(dv.ptr(R), n, dv.ptr(c), dv.ptr(y), None, s))
torch.cuda.synchronize()
e0 = torch.cuda.Event(True); e1 = torch.cuda.Event(True)
e0.record()
for _ in range(20):
    _lib.check(lib.itsk_trsv_pair(dv.ptr(R), n, dv.ptr(c), dv.ptr(y), None, s))
e1.record(); torch.cuda.synchronize()
print(f"n={n} trsv_pair {e0.elapsed_time(e1)/20*1e3:.1f} us")

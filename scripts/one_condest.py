import sys, os, ctypes
sys.path.insert(0, os.getcwd())
import torch
from paper_2311_04362_b200 import _lib
from paper_2311_04362_b200 import device as dv
lib = _lib.lib_for_device(0)
n = int(sys.argv[1])
g = torch.randn(3 * n, n, dtype=torch.float64, device="cuda")
r = torch.linalg.qr(g, mode="r")[1].contiguous()
v0 = torch.randn(n, dtype=torch.float64, device="cuda")
out = torch.empty(2, dtype=torch.float64, device="cuda")
ws = torch.empty(n * n, dtype=torch.float64, device="cuda")
_lib.check(lib.itsk_condest_ws(dv.ptr(r), n, dv.ptr(v0), dv.ptr(out), None, dv.ptr(ws), n * n, dv.stream_ptr()))
torch.cuda.synchronize()

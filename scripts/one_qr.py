import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2311_04362_b200 import _lib
from paper_2311_04362_b200 import device as dv
from paper_2311_04362_b200.linalg import qr_workspace
d, n1 = int(sys.argv[1]), int(sys.argv[2]); n = n1 - 1
lib = _lib.lib_for_device(0)
W = torch.randn(d, n1, dtype=torch.float64, device="cuda")
R = torch.empty(n, n, dtype=torch.float64, device="cuda"); z = torch.empty(n, dtype=torch.float64, device="cuda")
ws = qr_workspace(d, n, W.device)
_lib.check(lib.itsk_qr_aug(dv.ptr(W), d, n, n1, dv.ptr(R), dv.ptr(z), dv.ptr(ws), ws.numel(), dv.stream_ptr()))
torch.cuda.synchronize()
print("ok")

import sys, os, ctypes
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2311_04362_b200 import _lib
from paper_2311_04362_b200 import device as dv
from paper_2311_04362_b200.linalg import qr_workspace
d, n = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
lib = _lib.lib_for_device(0)
W0 = torch.randn(d, n + 1, dtype=torch.float64, device="cuda")
W = W0.clone(); R = torch.empty(n, n, dtype=torch.float64, device="cuda"); z = torch.empty(n, dtype=torch.float64, device="cuda")
ws = qr_workspace(d, n, W.device)
s = dv.stream_ptr()
def run():
    W.copy_(W0)
    _lib.check(lib.itsk_qr_aug(dv.ptr(W), d, n, n + 1, dv.ptr(R), dv.ptr(z), dv.ptr(ws), ws.numel(), s))
for _ in range(2): run()
torch.cuda.synchronize()
ts = []
for _ in range(reps):
    e0 = torch.cuda.Event(True); e1 = torch.cuda.Event(True)
    e0.record(); run(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
print(f"qr d={d} n={n}: {np.median(ts)*1e3:.1f} us")

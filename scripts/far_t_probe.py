"""Phase cycles of k_far_t (diagnostic build: python -c "from paper_2311_04362_b200 import build;
build.build(probe='farprobe')"): python scripts/far_t_probe.py d n"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2311_04362_b200 import _lib
from paper_2311_04362_b200 import device as dv
from paper_2311_04362_b200.linalg import qr_workspace

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = _lib.load(os.path.join(HERE, "paper_2311_04362_b200", "libitsk_b200_farprobe.so"))
lib.itsk_farprobe_read.argtypes = [ctypes.c_void_p]
d, n = int(sys.argv[1]), int(sys.argv[2])
ldw = (n + 2) // 2 * 2
W = torch.randn(d, ldw, dtype=torch.float64, device="cuda")
R = torch.empty(n, n, dtype=torch.float64, device="cuda")
z = torch.empty(n, dtype=torch.float64, device="cuda")
ws = qr_workspace(d, n, W.device)
_lib.check(lib.itsk_qr_aug(dv.ptr(W), d, n, ldw, dv.ptr(R), dv.ptr(z), dv.ptr(ws), ws.numel(), dv.stream_ptr()))
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 8)()
lib.itsk_farprobe_read(ctypes.addressof(buf))
names = ["load G", "P = T1 G", "all T_JJ", "-P T_JJ", "write T"]
tot = sum(buf[:5])
for i, nm in enumerate(names):
    print(f"{nm:10s} {buf[i] / 1e3:10.1f} kcycles  {100 * buf[i] / max(tot, 1):5.1f} %")

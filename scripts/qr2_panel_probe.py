"""Phase cycles of k_qr_panel, CTA 0 (diagnostic build: python -c "from
paper_2311_04362_b200 import build; build.build(probe='qr2_profile')"):
python scripts/qr2_panel_probe.py d n"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2311_04362_b200 import _lib
from paper_2311_04362_b200 import device as dv
from paper_2311_04362_b200.linalg import qr_workspace

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = _lib.load(os.path.join(HERE, "paper_2311_04362_b200", "libitsk_b200_qr2_profile.so"))
lib.itsk_qr2_profile_read.argtypes = [ctypes.c_void_p]
d, n = int(sys.argv[1]), int(sys.argv[2])
ldw = (n + 2) // 2 * 2
W = torch.randn(d, ldw, dtype=torch.float64, device="cuda")
R = torch.empty(n, n, dtype=torch.float64, device="cuda")
z = torch.empty(n, dtype=torch.float64, device="cuda")
ws = qr_workspace(d, n, W.device)
buf = (ctypes.c_ulonglong * 12)()
for rep in range(2):
    lib.itsk_qr2_profile_read(ctypes.addressof(buf))  # read and reset
    _lib.check(lib.itsk_qr_aug(dv.ptr(W), d, n, ldw, dv.ptr(R), dv.ptr(z), dv.ptr(ws), ws.numel(), dv.stream_ptr()))
    torch.cuda.synchronize()
lib.itsk_qr2_profile_read(ctypes.addressof(buf))
names = ["sweep", "warp reduce + sync", "record send", "cluster wait", "coef (pivot, tau)", "flush + sync",
         "G sum over cluster", "load panel", "write back", "G on DMMA", "cluster sync"]
npan = (n + 15) // 16
tot = sum(buf)
for i, nm in enumerate(names):
    print(f"{nm:20s} {buf[i] / npan / 1e3:8.2f} kcycles per panel  {100 * buf[i] / max(tot, 1):5.1f} %")
print(f"total {tot / npan / 1e3:.1f} kcycles per panel ({npan} panels)")

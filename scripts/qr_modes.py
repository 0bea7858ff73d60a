"""QR of the augmented sketch at the bench shapes: every itsk path (v2 = product,
v1 cluster, grid, tsqr) and cuSOLVER's geqrf via torch.linalg.qr (library
yardstick, R only) — device ms, median of 5."""
import ctypes, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2311_04362_b200 import _lib
from paper_2311_04362_b200 import device as dv
from paper_2311_04362_b200.linalg import qr_workspace

lib = _lib.lib_for_device(0)
shapes = [(4000, 201), (10000, 501), (24000, 2001)]


def t_med(fn, reps=5):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(True); e1 = torch.cuda.Event(True); e0.record(); fn(); e1.record()
        torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


for d, n1 in shapes:
    n = n1 - 1
    g = torch.Generator(device="cuda").manual_seed(d + n)
    W0 = torch.randn(d, n1, dtype=torch.float64, device="cuda", generator=g)
    W0 = W0 * torch.logspace(0, -8, n1, dtype=torch.float64, device="cuda")
    W = W0.clone(); R = torch.empty(n, n, dtype=torch.float64, device="cuda"); z = torch.empty(n, dtype=torch.float64, device="cuda")
    ws = qr_workspace(d, n, W.device)
    s = dv.stream_ptr()
    for mode in (os.environ.get("QRM_MODES", "v2,v1,grid,tsqr").split(",")):
        os.environ["ITSK_QR_MODE"] = mode
        def run():
            W.copy_(W0)
            _lib.check(lib.itsk_qr_aug(dv.ptr(W), d, n, n1, dv.ptr(R), dv.ptr(z), dv.ptr(ws), ws.numel(), s))
        try:
            run(); torch.cuda.synchronize()
            t = t_med(run) - t_med(lambda: W.copy_(W0))
            print(f"{d}x{n1} itsk {mode:5s} {t:8.3f} ms", flush=True)
        except Exception as e:
            print(f"{d}x{n1} itsk {mode:5s} n/a ({str(e)[:60]})", flush=True)
    os.environ.pop("ITSK_QR_MODE", None)
    torch.linalg.qr(W0, mode="r"); torch.cuda.synchronize()
    t = t_med(lambda: torch.linalg.qr(W0, mode="r"))
    print(f"{d}x{n1} cusolver geqrf (torch.linalg.qr mode=r) {t:8.3f} ms", flush=True)

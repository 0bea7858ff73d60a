"""condest (two TRSVs per Lanczos step) vs condest_ws (X = R^-1, matvecs), and the TRSV pair, vs n."""
import sys, os, ctypes
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2311_04362_b200 import _lib
from paper_2311_04362_b200 import device as dv
lib = _lib.lib_for_device(0)
dev = torch.device("cuda", 0)
for n in [int(v) for v in sys.argv[1:]]:
    g = torch.randn(3 * n, n, dtype=torch.float64, device=dev)
    r = torch.linalg.qr(g, mode="r")[1].contiguous()
    r = r * torch.sign(torch.diagonal(r))[:, None]
    v0 = torch.randn(n, dtype=torch.float64, device=dev)
    out = torch.empty(2, dtype=torch.float64, device=dev)
    nb = ctypes.c_int64(); lib.itsk_pack_upper_doubles(n, ctypes.byref(nb))
    rp = torch.empty(nb.value, dtype=torch.float64, device=dev)
    _lib.check(lib.itsk_pack_upper(dv.ptr(r), n, dv.ptr(rp), dv.stream_ptr()))
    ws = torch.empty(n * n, dtype=torch.float64, device=dev)
    c = torch.randn(n, dtype=torch.float64, device=dev); y = torch.empty_like(c)
    def T(fn, reps=3):
        fn(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(reps): fn()
        e1.record(); torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps
    t1 = T(lambda: _lib.check(lib.itsk_condest(dv.ptr(r), n, dv.ptr(v0), dv.ptr(out), dv.ptr(rp), dv.stream_ptr())))
    a = out[0].item()
    t2 = T(lambda: _lib.check(lib.itsk_condest_ws(dv.ptr(r), n, dv.ptr(v0), dv.ptr(out), dv.ptr(rp), dv.ptr(ws), n * n, dv.stream_ptr())))
    b = out[0].item()
    t3 = T(lambda: _lib.check(lib.itsk_trsv_pair(dv.ptr(r), n, dv.ptr(c), dv.ptr(y), None, dv.stream_ptr())))
    t4 = T(lambda: _lib.check(lib.itsk_normest(dv.ptr(r), n, dv.ptr(v0), 11, dv.ptr(out), dv.ptr(rp), dv.stream_ptr())))
    print(f"n={n}: condest {t1:.3f} ms  condest_ws {t2:.3f} ms (rel diff {abs(a-b)/a:.1e})  trsv_pair {t3:.3f} ms  normest {t4:.3f} ms")

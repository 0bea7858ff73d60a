"""CUDA-event timing of the TRSV pair R'y = c, R x = y: the one-CTA kernel
(itsk_trsv_pair) against the 16-CTA cluster kernel (itsk_trsv_pair_cl).
python scripts/micro_trsv_pair.py [n ...]"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2311_04362_b200  # noqa: F401
from paper_2311_04362_b200 import _lib
from paper_2311_04362_b200 import device as dv

dev = torch.device("cuda")
lib = dv.lib(dev)
for n in [int(v) for v in sys.argv[1:]] or [256, 500, 1000, 2000, 3000, 4096]:
    g = torch.Generator(device=dev).manual_seed(n)
    R = torch.triu(torch.randn(n, n, dtype=torch.float64, device=dev, generator=g)) / np.sqrt(n)
    R.diagonal().copy_(1.0 + torch.rand(n, dtype=torch.float64, device=dev, generator=g))
    nb = ctypes.c_int64()
    _lib.check(lib.itsk_pack_upper_doubles(n, ctypes.byref(nb)))
    Rp = torch.empty(nb.value, dtype=torch.float64, device=dev)
    _lib.check(lib.itsk_pack_upper(dv.ptr(R), n, dv.ptr(Rp), dv.stream_ptr()))
    c = torch.randn(n, dtype=torch.float64, device=dev, generator=g)
    d = torch.empty(n, dtype=torch.float64, device=dev)
    cs = torch.empty(n, dtype=torch.float64, device=dev)
    def one():
        cs.copy_(c)
        _lib.check(lib.itsk_trsv_pair(dv.ptr(R), n, dv.ptr(cs), dv.ptr(d), None, dv.stream_ptr()))
    def cl():
        _lib.check(lib.itsk_trsv_pair_cl(dv.ptr(R), dv.ptr(Rp), n, dv.ptr(c), dv.ptr(d), dv.stream_ptr()))
    out = {}
    for name, fn in (("one-CTA", one), ("cluster", cl)):
        for _ in range(3):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(50):
            fn()
        e1.record()
        torch.cuda.synchronize()
        out[name] = e0.elapsed_time(e1) / 50 * 1e3
    print(f"n={n:5d}  one-CTA {out['one-CTA']:8.1f} us (incl. 8n-byte copy)   cluster {out['cluster']:8.1f} us", flush=True)

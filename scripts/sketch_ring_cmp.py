"""Register gather vs cp.async ring sketch kernels (ITSK_SKETCH_RING) on C5-like
points and C2: device ms and GB/s of the algorithmic bytes 8 m (n+1)."""
import ctypes, json, os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2311_04362_b200 import _lib
from paper_2311_04362_b200 import device as dv
from paper_2311_04362_b200.embed import pcg_state

peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6500.0
lib = _lib.lib_for_device(0)
dev = torch.device("cuda")
s = int(torch.cuda.current_stream().cuda_stream)
words, h, pend = pcg_state(0)
pts = [(200000, 200, 4000, 8)]
for n in (100, 500, 2000):
    for dm in (4, 12, 20):
        for zeta in (4, 8, 16):
            m = 1 << 22 if n < 2000 else 1 << 20
            pts.append((m, n, dm * n, zeta))
print(f"{'m':>9s} {'n':>5s} {'d':>6s} {'zeta':>4s} {'gather ms':>10s} {'ring ms':>10s} {'gather GB/s':>11s} {'ring GB/s':>10s} {'best %peak':>10s}")
for m, n, d, zeta in pts:
    g = torch.Generator(device=dev).manual_seed(m + n)
    A = torch.randn(m, n, dtype=torch.float64, device=dev, generator=g)
    b = torch.randn(m, dtype=torch.float64, device=dev, generator=g)
    W = torch.empty(d, n + 1, dtype=torch.float64, device=dev)
    nnz = m * zeta
    rows = torch.empty(nnz, dtype=torch.int32, device=dev)
    neg = torch.empty(nnz, dtype=torch.uint8, device=dev)
    sk_ptr = torch.empty(d + 1, dtype=torch.int32, device=dev)
    sk_src = torch.empty(nnz, dtype=torch.int32, device=dev)
    nb = ctypes.c_int64()
    _lib.check(lib.itsk_pattern_workspace(d, m, zeta, ctypes.byref(nb)))
    ws = dv.workspace(nb.value, dev)
    _lib.check(lib.itsk_sparse_sign_pattern(d, m, zeta, words, h, pend, dv.ptr(rows), dv.ptr(neg),
                                            dv.ptr(sk_ptr), dv.ptr(sk_src), dv.ptr(ws), ws.numel(), s))
    res = {}
    outs = {}
    for ring in ("0", "1"):
        os.environ["ITSK_SKETCH_RING"] = ring
        fn = lambda: _lib.check(lib.itsk_sketch(dv.ptr(A), m, n, n, dv.ptr(b), dv.ptr(sk_ptr), dv.ptr(sk_src), d,
                                                zeta, dv.ptr(W), n + 1, s))
        fn(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(3):
            fn()
        e1.record(); torch.cuda.synchronize()
        res[ring] = e0.elapsed_time(e1) / 3
        outs[ring] = W.clone()
    assert torch.equal(outs["0"], outs["1"]), (m, n, d, zeta)
    gb = lambda t: 8 * m * (n + 1) / t / 1e6
    best = min(res.values())
    print(f"{m:9d} {n:5d} {d:6d} {zeta:4d} {res['0']:10.3f} {res['1']:10.3f} {gb(res['0']):11.0f} {gb(res['1']):10.0f} "
          f"{100 * gb(best) / peak:9.1f}%", flush=True)
    del A, b, W, rows, neg, sk_ptr, sk_src, ws, outs
    torch.cuda.empty_cache()

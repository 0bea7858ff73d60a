"""C5: sketch-only sweep (BASELINE configs[4]): S·[A|b] on seeded Gaussian fp64 A,
m = 2^20 .. 2^24, n in {100, 500, 2000}, d in {4n, 12n, 20n}, zeta in {4, 8, 16}.
Reports device ms of the pattern generation and of the sketch, and the sketch's
GB/s over the algorithmic bytes 8 m (n+1) (A and b read once) against the HBM
peak.  Points with A > 70 GB are skipped (m = 2^24 x n = 2000 is 268 GB).

    python scripts/sketch_sweep.py [out.txt]
"""
import ctypes, json, os, sys, time
sys.path.insert(0, os.getcwd())
import torch
from paper_2311_04362_b200 import _lib
from paper_2311_04362_b200 import device as dv
from paper_2311_04362_b200.embed import pcg_state

peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6650.0
lib = _lib.lib_for_device(0)
dev = torch.device("cuda")
s = int(torch.cuda.current_stream().cuda_stream)
words, h, pend = pcg_state(0)
lines = []


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


hdr = f"{'m':>9s} {'n':>5s} {'d':>6s} {'zeta':>4s} {'pattern ms':>10s} {'sketch ms':>10s} {'GB/s':>7s} {'%peak':>6s}"
print(hdr, flush=True)
lines.append(hdr)
for n in (100, 500, 2000):
    for lm in (20, 22, 24):
        m = 1 << lm
        if 8 * m * n > 70e9:
            continue
        g = torch.Generator(device=dev).manual_seed(lm * 7 + n)
        A = torch.randn(m, n, dtype=torch.float64, device=dev, generator=g)
        b = torch.randn(m, dtype=torch.float64, device=dev, generator=g)
        for dm in (4, 12, 20):
            d = dm * n
            W = torch.empty(d, n + 1, dtype=torch.float64, device=dev)
            for zeta in (4, 8, 16):
                nnz = m * zeta
                rows = torch.empty(nnz, dtype=torch.int32, device=dev)
                neg = torch.empty(nnz, dtype=torch.uint8, device=dev)
                sk_ptr = torch.empty(d + 1, dtype=torch.int32, device=dev)
                sk_src = torch.empty(nnz, dtype=torch.int32, device=dev)
                nb = ctypes.c_int64()
                _lib.check(lib.itsk_pattern_workspace(d, m, zeta, ctypes.byref(nb)))
                ws = dv.workspace(nb.value, dev)

                def pattern():
                    _lib.check(lib.itsk_sparse_sign_pattern(d, m, zeta, words, h, pend, dv.ptr(rows), dv.ptr(neg),
                                                            dv.ptr(sk_ptr), dv.ptr(sk_src), dv.ptr(ws), ws.numel(), s))

                def sketch():
                    _lib.check(lib.itsk_sketch(dv.ptr(A), m, n, n, dv.ptr(b), dv.ptr(sk_ptr), dv.ptr(sk_src), d, zeta,
                                               dv.ptr(W), n + 1, s))

                reps = 3 if 8 * m * n < 8e9 else 1
                tp = timed(pattern, reps)
                ts = timed(sketch, reps)
                gbs = 8 * m * (n + 1) / ts / 1e6
                ln = f"{m:9d} {n:5d} {d:6d} {zeta:4d} {tp:10.3f} {ts:10.3f} {gbs:7.0f} {100 * gbs / peak:5.1f}%"
                print(ln, flush=True)
                lines.append(ln)
                del rows, neg, sk_ptr, sk_src, ws
            del W
        del A, b
        torch.cuda.empty_cache()
if len(sys.argv) > 1:
    open(sys.argv[1], "w").write("\n".join(lines) + "\n")

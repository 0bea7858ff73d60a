"""Phase cycles of the v2 panel kernel (CTA 0), libqr2prof.so built with -DITSK_QR2_PROFILE:
  cd paper_2311_04362_b200/csrc && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \\
    -Xcompiler -fPIC --expt-relaxed-constexpr -I. -I../../include -DITSK_QR2_PROFILE -shared \\
    -o ../../scripts/bw/libqr2prof.so capi.cu qr.cu qr2.cu qr_tsqr.cu trsv.cu pass.cu loop.cu pattern.cu sketch.cu \\
    -lcudart_static -lrt -ldl -lpthread"""
import ctypes, sys, os, torch
lib = ctypes.CDLL(os.path.abspath(sys.argv[3] if len(sys.argv) > 3 else "scripts/bw/libqr2prof.so"))
d, n = int(sys.argv[1]), int(sys.argv[2])
W0 = torch.randn(d, n + 1, dtype=torch.float64, device="cuda"); W = W0.clone()
R = torch.empty(n, n, dtype=torch.float64, device="cuda"); z = torch.empty(n, dtype=torch.float64, device="cuda")
nb = ctypes.c_int64(); lib.itsk_qr_workspace(ctypes.c_int64(d), ctypes.c_int64(n), ctypes.byref(nb))
ws = torch.empty(nb.value, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream().cuda_stream
P = ctypes.c_void_p
out = (ctypes.c_ulonglong * 8)()
for it in range(2):
    W.copy_(W0); torch.cuda.synchronize()
    lib.itsk_qr2_profile_read(out)
    rc = lib.itsk_qr_aug(P(W.data_ptr()), ctypes.c_int64(d), ctypes.c_int64(n), ctypes.c_int64(n + 1), P(R.data_ptr()), P(z.data_ptr()), P(ws.data_ptr()), ctypes.c_int64(ws.numel()), P(s))
    torch.cuda.synchronize()
    lib.itsk_qr2_profile_read(out)
names = ["sweep", "syncthreads", "reduce+push", "cluster.sync", "coeffs", "(end loop)", "writeback+G+T", "panel load"]
tot = sum(out[i] for i in range(8))
for i, nm in enumerate(names): print(f"{nm:14s} {out[i]:10d} cycles {100*out[i]/max(tot,1):5.1f}%  per col {out[i]/n:8.0f}")
print("total", tot, "cycles =", tot / 1.9e3, "us", "rc", rc)

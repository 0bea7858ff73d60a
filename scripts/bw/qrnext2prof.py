"""Phase cycles of k_qr_next2 (CTA 0, summed over launches), lib built with -DITSK_QRNEXT_PROBE:
  cd paper_2311_04362_b200/csrc && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \\
    -Xcompiler -fPIC --expt-relaxed-constexpr -I. -I../../include -DITSK_QRNEXT_PROBE -shared \\
    -o ../../scripts/bw/libqrnext.so capi.cu qr.cu qr2.cu qr_far.cu qr_tsqr.cu trsv.cu pass.cu loop.cu \\
    pattern.cu sketch.cu sparse.cu -lcudart_static -lrt -ldl -lpthread"""
import ctypes, sys, os, torch
lib = ctypes.CDLL(os.path.abspath(sys.argv[3] if len(sys.argv) > 3 else "scripts/bw/libqrnext.so"))
d, n = int(sys.argv[1]), int(sys.argv[2])
W0 = torch.randn(d, n + 1, dtype=torch.float64, device="cuda"); W = W0.clone()
R = torch.empty(n, n, dtype=torch.float64, device="cuda"); z = torch.empty(n, dtype=torch.float64, device="cuda")
nb = ctypes.c_int64(); lib.itsk_qr_workspace(ctypes.c_int64(d), ctypes.c_int64(n), ctypes.byref(nb))
ws = torch.empty(nb.value, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream().cuda_stream
P = ctypes.c_void_p
a = (ctypes.c_ulonglong * 8)(); b = (ctypes.c_ulonglong * 8)()
for it in range(3):
    W.copy_(W0); torch.cuda.synchronize()
    lib.itsk_qrnext_profile_read(a)
    rc = lib.itsk_qr_aug(P(W.data_ptr()), ctypes.c_int64(d), ctypes.c_int64(n), ctypes.c_int64(n + 1), P(R.data_ptr()), P(z.data_ptr()), P(ws.data_ptr()), ctypes.c_int64(ws.numel()), P(s))
    torch.cuda.synchronize()
    lib.itsk_qrnext_profile_read(b)
names = ["pass1 (Y partial)", "cluster.sync", "cluster reduce", "Z", "pass2 (B -= VZ)", "final cluster.sync"]
launches = 110 if n == 2000 else 1
for i, nm in enumerate(names): print(f"{nm:20s} {(b[i]-a[i])/launches:10.0f} cycles per launch")

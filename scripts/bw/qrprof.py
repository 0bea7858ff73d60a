import ctypes, sys, os, numpy as np, torch
sys.path.insert(0, os.getcwd())
lib = ctypes.CDLL(os.path.abspath("scripts/bw/libqrprof.so"))
d, n = int(sys.argv[1]), int(sys.argv[2])
W0 = torch.randn(d, n + 1, dtype=torch.float64, device="cuda"); W = W0.clone()
R = torch.empty(n, n, dtype=torch.float64, device="cuda"); z = torch.empty(n, dtype=torch.float64, device="cuda")
nb = ctypes.c_int64(); lib.itsk_qr_workspace(ctypes.c_int64(d), ctypes.c_int64(n), ctypes.byref(nb))
ws = torch.empty(nb.value, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream().cuda_stream
P = ctypes.c_void_p
for it in range(2):
    W.copy_(W0); torch.cuda.synchronize()
    rc = lib.itsk_qr_aug(P(W.data_ptr()), ctypes.c_int64(d), ctypes.c_int64(n), ctypes.c_int64(n + 1), P(R.data_ptr()), P(z.data_ptr()), P(ws.data_ptr()), ctypes.c_int64(ws.numel()), P(s))
    out = (ctypes.c_ulonglong * 16)(); lib.itsk_qr_profile_read(out)
names = ["col-start", "partials", "sync", "rec-read", "scalars", "update", "panel-wb", "GY", "sync", "G/T/Z", "sync", "W-update"]
tot = sum(out[i] for i in range(12))
for i, nm in enumerate(names): print(f"{nm:10s} {out[i]:10d} cycles {100*out[i]/tot:5.1f}%")
print("total", tot, "cycles =", tot / 1.9e3, "us", "rc", rc)

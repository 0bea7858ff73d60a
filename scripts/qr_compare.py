"""R from the v2 (panel/update split) QR vs the v1 single-kernel QR and LAPACK."""
import os, sys, subprocess, json
sys.path.insert(0, os.getcwd())
import numpy as np, torch
shapes = [(20, 5), (300, 40), (4000, 201), (10000, 501), (24000, 2001)] if len(sys.argv) < 2 else [tuple(map(int, a.split("x"))) for a in sys.argv[1:]]
if os.environ.get("QRC_CHILD"):
    from paper_2311_04362_b200 import _lib
    from paper_2311_04362_b200 import device as dv
    from paper_2311_04362_b200.linalg import qr_workspace
    lib = _lib.lib_for_device(0)
    for d, n1 in shapes:
        n = n1 - 1
        g = torch.Generator(device="cuda").manual_seed(d + n)
        W0 = torch.randn(d, n1, dtype=torch.float64, device="cuda", generator=g)
        W0 = W0 * torch.logspace(0, -8, n1, dtype=torch.float64, device="cuda")
        W = W0.clone(); R = torch.empty(n, n, dtype=torch.float64, device="cuda"); z = torch.empty(n, dtype=torch.float64, device="cuda")
        ws = qr_workspace(d, n, W.device)
        s = dv.stream_ptr()
        _lib.check(lib.itsk_qr_aug(dv.ptr(W), d, n, n1, dv.ptr(R), dv.ptr(z), dv.ptr(ws), ws.numel(), s))
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            W.copy_(W0); torch.cuda.synchronize()
            e0 = torch.cuda.Event(True); e1 = torch.cuda.Event(True); e0.record()
            _lib.check(lib.itsk_qr_aug(dv.ptr(W), d, n, n1, dv.ptr(R), dv.ptr(z), dv.ptr(ws), ws.numel(), s))
            e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
        np.save(f"/tmp/qr_{os.environ.get('ITSK_QR_MODE','v2')}_{d}x{n1}.npy", np.concatenate([R.cpu().numpy().ravel(), z.cpu().numpy()]))
        if d * n1 < 3e6:
            np.save(f"/tmp/qr_in_{d}x{n1}.npy", W0.cpu().numpy())
        print(f"{os.environ.get('ITSK_QR_MODE','v2')} {d}x{n1}: {np.median(ts)*1e3:.1f} us", flush=True)
else:
    for mode in ["v2", "v1"]:
        env = dict(os.environ, QRC_CHILD="1", ITSK_QR_MODE=mode)
        subprocess.run([sys.executable, __file__] + sys.argv[1:], env=env, check=True)
    for d, n1 in shapes:
        n = n1 - 1
        a = np.load(f"/tmp/qr_v2_{d}x{n1}.npy"); b = np.load(f"/tmp/qr_v1_{d}x{n1}.npy")
        R2, R1 = a[:n*n].reshape(n, n), b[:n*n].reshape(n, n)
        rel = np.linalg.norm(R2 - R1) / np.linalg.norm(R1)
        zr = np.linalg.norm(a[n*n:] - b[n*n:]) / np.linalg.norm(b[n*n:])
        msg = f"{d}x{n1}: ||R2-R1||/||R1|| = {rel:.2e}  z rel {zr:.2e}"
        if os.path.exists(f"/tmp/qr_in_{d}x{n1}.npy"):
            W0 = np.load(f"/tmp/qr_in_{d}x{n1}.npy")
            Rl = np.linalg.qr(W0[:, :n], mode="r"); Rl = Rl * np.sign(np.diag(Rl))[:, None]
            msg += f"  vs LAPACK {np.linalg.norm(R2 - Rl) / np.linalg.norm(Rl):.2e} (v1 {np.linalg.norm(R1 - Rl) / np.linalg.norm(Rl):.2e})"
        print(msg)

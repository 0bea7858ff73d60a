import ctypes, sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2311_04362_b200 as pkg
from paper_2311_04362_b200 import _lib
from paper_2311_04362_b200 import device as dv
for n, kappa, ill in [(2047, 1e6, True), (2047, 1e6, False), (2048, 1e6, True), (777, 1e12, True), (4096, 1e4, False)]:
    rng = np.random.default_rng(n)
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    s = kappa ** (-np.arange(n) / (n - 1))
    r = np.linalg.qr((q * s) @ np.linalg.qr(rng.standard_normal((n, n)))[0].T, mode="r")
    r = r * np.sign(np.diag(r))[:, None]
    if ill:
        for b0 in (64, 32 * (n // 64)):
            r[b0 + 5, b0 + 5] *= 1e-6
    c = rng.standard_normal(n)
    dev = torch.device("cuda")
    R = torch.from_numpy(np.ascontiguousarray(r)).to(dev)
    nb = ctypes.c_int64(); lib = dv.lib(dev)
    _lib.check(lib.itsk_pack_upper_doubles(n, ctypes.byref(nb)))
    Rp = torch.empty(nb.value, dtype=torch.float64, device=dev)
    _lib.check(lib.itsk_pack_upper(dv.ptr(R), n, dv.ptr(Rp), dv.stream_ptr()))
    ct = torch.from_numpy(c).to(dev)
    outs = []
    for rep in range(5):
        d = torch.full((n,), float("nan"), dtype=torch.float64, device=dev)
        _lib.check(lib.itsk_trsv_pair_cl(dv.ptr(R), dv.ptr(Rp), n, dv.ptr(ct), dv.ptr(d), dv.stream_ptr()))
        outs.append(d.cpu().numpy())
    nf = [int((~np.isfinite(o)).sum()) for o in outs]
    diffs = [np.nonzero(o != outs[0])[0][:8].tolist() for o in outs[1:]]
    import scipy.linalg as sl
    ref = sl.solve_triangular(r, sl.solve_triangular(r, c, trans="T"))
    print(n, kappa, ill, "nonfinite", nf, "diff idx", diffs, "relerr", [float(np.linalg.norm(o - ref) / np.linalg.norm(ref)) for o in outs[:2]], flush=True)

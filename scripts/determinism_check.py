"""Bitwise run-to-run check of the QR and the full solve at a given shape:
    python scripts/determinism_check.py d n [m]  -> prints digests (compare across processes / env knobs)"""
import hashlib, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2311_04362_b200 as itsk
from paper_2311_04362_b200 import _lib
from paper_2311_04362_b200 import device as dv
from paper_2311_04362_b200.linalg import qr_workspace

d, n = int(sys.argv[1]), int(sys.argv[2])
m = int(sys.argv[3]) if len(sys.argv) > 3 else 0
lib = _lib.lib_for_device(0)
g = torch.Generator(device="cuda").manual_seed(7)
W0 = torch.randn(d, n + 1, dtype=torch.float64, device="cuda", generator=g)
W0 *= torch.logspace(0, -8, n + 1, dtype=torch.float64, device="cuda")
ws = qr_workspace(d, n, W0.device)
dig = []
for rep in range(3):
    W = W0.clone()
    R = torch.empty(n, n, dtype=torch.float64, device="cuda")
    z = torch.empty(n, dtype=torch.float64, device="cuda")
    _lib.check(lib.itsk_qr_aug(dv.ptr(W), d, n, n + 1, dv.ptr(R), dv.ptr(z), dv.ptr(ws), ws.numel(), dv.stream_ptr()))
    torch.cuda.synchronize()
    dig.append(hashlib.sha256(R.cpu().numpy().tobytes() + z.cpu().numpy().tobytes()).hexdigest()[:16])
print(f"qr {d}x{n} digests {dig} env_lookahead={os.environ.get('ITSK_QR_LOOKAHEAD', '1')}", flush=True)
if m:
    from paper_2311_04362_b200.instances import gen_randsvd_device
    p = gen_randsvd_device(m, n, 1e8, 1e-6, 0)
    sd = []
    for rep in range(3):
        res = itsk.iterative_sketching(p.a, p.b, itsk.SolverConfig(d=d, variant="momentum"), p.truth, residuals="all")
        sd.append((hashlib.sha256(res.solution.tobytes()).hexdigest()[:16], res.iterations, f"{res.trace.fe[-1]:.6e}"))
    print(f"solve m={m} digests {sd}", flush=True)

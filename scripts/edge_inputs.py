"""Probe of input forms on the GPU box: Fortran-ordered / strided / row-sliced / float32 / integer A, list b,
non-contiguous device tensors (all must give the contiguous float64 result bit for bit or to rounding),
and malformed inputs (wrong length, 1-D A, m < n, NaN).  python scripts/edge_inputs.py"""
import numpy as np, torch, sys
sys.path.insert(0, "/root/repo")
import paper_2311_04362_b200 as itsk
from oracle import itsketch_oracle as orc
a, b, t = orc.gen_randsvd(4000, 50, 1e6, 1e-6, 0)
cfg = itsk.SolverConfig(d=1000)
ref = itsk.iterative_sketching(a, b, cfg).solution
for name, aa, bb in [("fortran", np.asfortranarray(a), b), ("strided", np.ascontiguousarray(np.hstack([a, a]))[:, :50], b),
                     ("rowslice", np.vstack([a, a])[:4000], b), ("list-b", a, list(b)), ("neg-stride", a[::-1][::-1], b),
                     ("torch-noncontig", torch.from_numpy(np.asfortranarray(a)).cuda(), torch.from_numpy(b).cuda())]:
    try:
        x = itsk.iterative_sketching(aa, bb, cfg).solution
        x = x.cpu().numpy() if isinstance(x, torch.Tensor) else x
        print(name, "ok", np.array_equal(x, ref), float(np.linalg.norm(x - ref) / np.linalg.norm(ref)))
    except Exception as e:
        print(name, "ERR", type(e).__name__, str(e)[:120])
for name, aa in [("float32", a.astype(np.float32)), ("int", np.round(a * 1e3).astype(np.int64))]:
    try:
        x = itsk.iterative_sketching(aa, b, cfg).solution
        xr, _ = orc.iterative_sketching(np.asarray(aa, dtype=float), b, orc.Config(d=1000))
        print(name, "ok", float(np.linalg.norm(x - xr) / np.linalg.norm(xr)))
    except Exception as e:
        print(name, "ERR", type(e).__name__, str(e)[:120])
for name, aa, bb in [("b-wrong-len", a, b[:-1]), ("a-1d", a[:, 0], b), ("wide", a[:40], b[:40]), ("nan", np.where(np.arange(a.size).reshape(a.shape) == 7, np.nan, a), b)]:
    try:
        r = itsk.iterative_sketching(aa, bb, itsk.SolverConfig(d=1000 if name != "wide" else 60))
        print(name, "returned", r.trace.stop_reason, r.iterations)
    except Exception as e:
        print(name, "ERR", type(e).__name__, str(e)[:120])

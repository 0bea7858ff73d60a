"""A/B of sketch kernel variants at one shape (same bits; the first variant is the bitwise reference):
    python scripts/sketch_sweep_ab.py [m n d zeta reps] [variant ...]
variant = an ITSK_SKETCH_SWCL value (0: 128-column panels, 2: 64-column panels) or a comma-separated list of
NAME=value pairs setting ITSK_SKETCH_<NAME> (SWEEP, SWCL, DRIFT, DIRECT, RING, GCPL, UNR), e.g. "DIRECT=0,SWCL=0".
Settings persist from one variant to the next: name every knob a comparison depends on."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2311_04362_b200 as itsk
m, n, d, zeta = (int(v) for v in sys.argv[1:5]) if len(sys.argv) > 4 else (4000000, 2000, 24000, 8)
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 4
shapes = [v for v in sys.argv[6:]] or ["0", "2"]
g = torch.Generator(device="cuda").manual_seed(0)
A = torch.randn(m, n, dtype=torch.float64, device="cuda", generator=g)
b = torch.randn(m, dtype=torch.float64, device="cuda", generator=g)
s = itsk.sparse_sign_new(d, m, zeta, 0)
ref = None
for sh in shapes:
    for tok in sh.split(","):  # "5" = shape, or NAME=value[,NAME=value] (suffix of ITSK_SKETCH_)
        key, _, val = tok.partition("=")
        if val:
            os.environ["ITSK_SKETCH_" + key] = val
        else:
            os.environ["ITSK_SKETCH_SWCL"] = tok
    ts = []
    for r in range(reps):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        w = s.apply_dense(A, b)
        torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    same = "" if ref is None else ("  bitwise equal" if torch.equal(w, ref) else "  DIFFERS")
    if ref is None:
        ref = w.clone()
    print(f"shape {sh}: " + " / ".join(f"{1e3 * t:.2f}" for t in ts) + f" ms{same}", flush=True)

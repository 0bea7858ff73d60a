"""Critical path of the refinement loop from %globaltimer stamps (diagnostic
build: python -m paper_2311_04362_b200.build --timeline).

Per iteration i (slot 0 = the begin pass + tail):
  pass   first CTA start -> last CTA end of streaming -> end of the reduction
  tail   entry -> dependency satisfied -> control -> R'y=c -> Rx=y -> end
and the gaps between them (us).  Usage: python scripts/loop_timeline.py [c2|c3] [variant]
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2311_04362_b200 import _lib  # noqa: E402

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = _lib.load(os.path.join(HERE, "paper_2311_04362_b200", "libitsk_b200_timeline.so"))
lib.itsk_pass_timeline_read.argtypes = [ctypes.c_void_p]
lib.itsk_tail_timeline_read.argtypes = [ctypes.c_void_p]

import paper_2311_04362_b200 as itsk  # noqa: E402
from bench import CONFIGS, make_problem  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
variant = sys.argv[2] if len(sys.argv) > 2 else "basic"
m, n, kappa, beta, d, zeta = CONFIGS[name]
p, _, _ = make_problem(name, 0)
dev = torch.device("cuda")
at = p.a if isinstance(p.a, torch.Tensor) else torch.from_numpy(p.a).to(dev)
bt = p.b if isinstance(p.b, torch.Tensor) else torch.from_numpy(p.b).to(dev)
cfg = itsk.SolverConfig(d=d, zeta=zeta, variant=variant)
P = np.zeros((64, 4), dtype=np.uint64)
T = np.zeros((64, 8), dtype=np.uint64)
for rep in range(4):
    res = itsk.iterative_sketching(at, bt, cfg, residuals="all")
    torch.cuda.synchronize()
    lib.itsk_pass_timeline_read(P.ctypes.data)
    lib.itsk_tail_timeline_read(T.ctypes.data)
K = res.iterations + 1
t0 = int(P[0, 0])


def us(x):
    return (int(x) - t0) / 1000.0


print(f"{name} {variant}: {res.iterations} iterations, stop {res.trace.stop_reason}")
print(f"{'slot':>4} {'p.start':>9} {'p.stream':>9} {'p.end':>9} {'t.wait':>9} {'t.ctl':>8} {'t.Rty':>8} "
      f"{'t.Rx':>8} {'t.end':>8} | {'pass':>7} {'reduce':>7} {'gap':>6} {'ctl':>6} {'Rty':>6} {'Rx':>6} {'upd':>6}")
rows = []
for i in range(K):
    ps, pe1, pe2 = us(P[i, 0]), us(P[i, 1]), us(P[i, 2])
    tw, tc, t1, t2, te = (us(T[i, k]) for k in (1, 2, 3, 4, 5))
    r = (pe1 - ps, pe2 - pe1, tw - pe2, tc - tw, t1 - tc, t2 - t1, te - t2)
    rows.append(r)
    print(f"{i:4d} {ps:9.1f} {pe1:9.1f} {pe2:9.1f} {tw:9.1f} {tc:8.1f} {t1:8.1f} {t2:8.1f} {te:8.1f} | "
          + " ".join(f"{v:6.1f}" for v in r))
med = np.median(np.array(rows[1:-1]), axis=0)
print("median (slots 1..K-2): pass %.1f reduce %.1f gap %.1f ctl %.1f Rty %.1f Rx %.1f upd %.1f us" % tuple(med))
print(f"iteration period (tail end to tail end): "
      f"{np.median(np.diff([us(T[i, 5]) for i in range(1, K - 1)])):.1f} us")

"""Per golden solve case: the B200 run's final FE/RE against the reference's
own (tests/golden/solves.npz) — which cases meet the strict north-star bar
(FE, RE <= 2x the reference's) and by what ratio.
    python scripts/strict_bar.py > profiles/<round>_strict_bar.txt"""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2311_04362_b200 as pkg
from oracle import itsketch_oracle as orc

g = np.load(os.path.join(ROOT, "tests", "golden", "solves.npz"))
names = ["c1_basic", "c1_damped", "c1_momentum", "c1_seed1", "c3like", "bitwise", "consistent", "extra3",
         "zero_init", "be_direct", "be_fast", "diverge", "maxit0", "eps_override", "c4proxy_mom"]
print(f"{'case':14s} {'stop':>16s} {'it':>4s} {'ref':>4s} {'FE':>10s} {'FE_ref':>10s} {'ratio':>6s} "
      f"{'RE':>10s} {'RE_ref':>10s} {'ratio':>6s} strict")
for name in names:
    m, n, kappa, beta, seed = g[f"{name}_problem"]
    a, b, truth = orc.gen_randsvd(int(m), int(n), kappa, beta, int(seed))
    cfgd = json.loads(str(g[f"{name}_config"]))
    t = pkg.Truth(x=truth.x, r=truth.r, kappa=truth.kappa, beta=truth.beta)
    res = pkg.iterative_sketching(a, b, pkg.SolverConfig(**cfgd), t)
    fe, re = res.trace.fe[-1], res.trace.re[-1]
    fr, rr = float(g[f"{name}_fe"][-1]), float(g[f"{name}_re"][-1])
    ok = fe <= 2 * fr + 4 * 2.0**-53 and re <= 2 * rr + 4 * 2.0**-53
    print(f"{name:14s} {res.trace.stop_reason:>16s} {res.iterations:4d} {len(g[f'{name}_iterates']) - 1:4d} "
          f"{fe:10.3e} {fr:10.3e} {fe / max(fr, 1e-300):6.2f} {re:10.3e} {rr:10.3e} {re / max(rr, 1e-300):6.2f} "
          f"{'yes' if ok else 'NO'}")

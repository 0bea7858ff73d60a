"""Random small configurations through the drop-in and the CPU oracle (shapes, sketch sizes, zeta, variants,
conditioning): reports exceptions raised on one side only, different stop reasons, and final errors beyond the
2x bar.  python scripts/fuzz_configs.py [count] [seed]"""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2311_04362_b200 as itsk
from oracle import itsketch_oracle as orc

count = int(sys.argv[1]) if len(sys.argv) > 1 else 40
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
U = 2.0 ** -53
bad = 0
for t in range(count):
    n = int(rng.integers(1, 300))
    m = int(rng.integers(n + 1, 6000))
    d = int(rng.integers(n, 8 * n + 2))
    zeta = int(rng.integers(1, min(d, 12) + 1))
    variant = str(rng.choice(["basic", "damped", "momentum"]))
    kappa = float(10.0 ** rng.integers(0, 12))
    beta = float(rng.choice([0.0, 1e-12, 1e-6, 1e-2]))
    seed = int(rng.integers(0, 100))
    max_iters = int(rng.choice([0, 1, 7, 50]))
    init = str(rng.choice(["sketch_and_solve", "zero"]))
    tag = f"m={m} n={n} d={d} zeta={zeta} {variant} kappa={kappa:.0e} beta={beta:.0e} seed={seed} max_iters={max_iters} {init}"
    try:
        a, b, tr_ = orc.gen_randsvd(m, n, max(kappa, 1.0), beta, seed) if n > 1 else (None, None, None)
        if a is None:
            a = rng.standard_normal((m, 1)); x = np.ones(1); b = a @ x
            tr_ = None
    except Exception as e:  # noqa: BLE001
        print("gen:", tag, type(e).__name__, e); continue
    r_o = r_d = e_o = e_d = None
    try:
        r_o = orc.iterative_sketching(a, b, orc.Config(d=d, zeta=zeta, variant=variant, rng_seed=seed,
                                                       max_iters=max_iters, init=init), tr_)
    except Exception as e:  # noqa: BLE001
        e_o = type(e).__name__
    try:
        truth = None if tr_ is None else itsk.Truth(x=tr_.x, r=tr_.r, kappa=tr_.kappa, beta=tr_.beta)
        r_d = itsk.iterative_sketching(a, b, itsk.SolverConfig(d=d, zeta=zeta, variant=variant, rng_seed=seed,
                                                               max_iters=max_iters, init=init), truth)
    except Exception as e:  # noqa: BLE001
        e_d = type(e).__name__ + ": " + str(e)[:80]
    if e_o or e_d:
        same = (e_o is not None) and (e_d is not None) and e_d.startswith(e_o)
        print(("ok   " if same else "DIFF ") + tag, "oracle:", e_o, "| device:", e_d)
        bad += 0 if same else 1
        continue
    x_o, t_o = r_o
    it_o = len(t_o.iterates) - 1
    msg = []
    if t_o.stop_reason != r_d.trace.stop_reason:
        msg.append(f"stop {r_d.trace.stop_reason} vs {t_o.stop_reason}")
    if abs(r_d.iterations - it_o) > max(3, 0.15 * it_o):
        msg.append(f"iters {r_d.iterations} vs {it_o}")
    if tr_ is not None and t_o.fe and np.isfinite(t_o.fe[-1]) and t_o.stop_reason != "diverged":
        if r_d.trace.fe[-1] > 2 * t_o.fe[-1] + 10 * kappa * U:
            msg.append(f"fe {r_d.trace.fe[-1]:.2e} vs {t_o.fe[-1]:.2e}")
    print(("ok   " if not msg else "DIFF ") + tag + (" :: " + "; ".join(msg) if msg else f" :: {t_o.stop_reason} {it_o}"), flush=True)
    bad += 1 if msg else 0
print(f"{bad} differences in {count} configurations")

"""Random sparse instances (gen_sparse and random CSR with empty rows / columns clipped away) through the
drop-in's CSR path and the CPU oracle: exceptions, stop reasons, final residual norms.
python scripts/fuzz_sparse.py [count] [seed]"""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import scipy.sparse as sp
import paper_2311_04362_b200 as itsk
from oracle import itsketch_oracle as orc

count = int(sys.argv[1]) if len(sys.argv) > 1 else 30
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
bad = 0
for t in range(count):
    n = int(rng.integers(2, 200))
    m = int(rng.integers(4 * n, 40 * n + 50))
    d = int(rng.integers(4 * n, 20 * n))
    variant = str(rng.choice(["basic", "damped", "momentum"]))
    seed = int(rng.integers(0, 50))
    fmt = str(rng.choice(["csr", "csc", "coo"]))
    if rng.random() < 0.5:
        p = itsk.gen_sparse(m, n, seed)
        a, b = p.a.asformat(fmt), p.b
    else:
        a = sp.random(m, n, density=float(rng.choice([0.01, 0.05, 0.3])), random_state=rng, format=fmt)
        a = a + sp.eye(m, n, format=fmt) * 0.5  # full column rank
        b = rng.standard_normal(m)
    tag = f"m={m} n={n} d={d} {variant} seed={seed} {fmt} nnz={a.nnz}"
    e_o = e_d = None
    try:
        x_o, t_o = orc.iterative_sketching(a.tocsr(), b, orc.Config(d=d, variant=variant, rng_seed=seed))
    except Exception as e:  # noqa: BLE001
        e_o = type(e).__name__
    try:
        r_d = itsk.iterative_sketching(a, b, itsk.SolverConfig(d=d, variant=variant, rng_seed=seed))
    except Exception as e:  # noqa: BLE001
        e_d = type(e).__name__ + ": " + str(e)[:80]
    if e_o or e_d:
        same = (e_o is not None) and (e_d is not None) and e_d.startswith(e_o)
        print(("ok   " if same else "DIFF ") + tag, "oracle:", e_o, "| device:", e_d, flush=True)
        bad += 0 if same else 1
        continue
    it_o = len(t_o.iterates) - 1
    msg = []
    if t_o.stop_reason != r_d.trace.stop_reason:
        msg.append(f"stop {r_d.trace.stop_reason} vs {t_o.stop_reason}")
    if abs(r_d.iterations - it_o) > max(3, 0.15 * it_o):
        msg.append(f"iters {r_d.iterations} vs {it_o}")
    rn_o = np.linalg.norm(b - a @ x_o)
    rn_d = np.linalg.norm(b - a @ r_d.solution)
    if t_o.stop_reason != "diverged" and rn_d > rn_o * (1 + 1e-8) + 1e-12:
        msg.append(f"residual {rn_d:.6e} vs {rn_o:.6e}")
    print(("ok   " if not msg else "DIFF ") + tag + (" :: " + "; ".join(msg) if msg else f" :: {t_o.stop_reason} {it_o}"), flush=True)
    bad += 1 if msg else 0
print(f"{bad} differences in {count} configurations")

"""C4 full-size parity run (4e6 x 2000, kappa 1e8, beta 1e-6, d = 12n, zeta 8):
the device-built instance solved by the B200 path and, on the same bytes
copied to the host, by the CPU oracle.  Writes profiles/c4_parity_<variant>.json.

    python scripts/c4_parity.py [variant] [seed]
"""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2311_04362_b200 as itsk
from paper_2311_04362_b200.instances import gen_randsvd_device
from oracle import itsketch_oracle as orc

variant = sys.argv[1] if len(sys.argv) > 1 else "momentum"
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 0
residuals = sys.argv[3] if len(sys.argv) > 3 else "all"  # "all": estimates deferred beside the loop
m, n, kappa, beta, d = 4_000_000, 2000, 1e8, 1e-6, 24000
U = 2.0 ** -53
t0 = time.time()
p = gen_randsvd_device(m, n, kappa, beta, seed)
torch.cuda.synchronize()
t_gen = time.time() - t0
cfg = itsk.SolverConfig(d=d, variant=variant, rng_seed=seed)
res = itsk.iterative_sketching(p.a, p.b, cfg, p.truth, residuals=residuals)
torch.cuda.synchronize()
t0 = time.time()
res = itsk.iterative_sketching(p.a, p.b, cfg, p.truth, residuals=residuals)
torch.cuda.synchronize()
t_gpu = time.time() - t0
out = {"config": "c4", "residuals": residuals, "m": m, "n": n, "kappa": kappa, "beta": beta, "d": d, "zeta": 8, "variant": variant,
       "seed": seed, "generate_s": t_gen, "gpu_solve_wall_s": t_gpu,
       "gpu": {"iterations": res.iterations, "stop": res.trace.stop_reason, "fe": res.trace.fe[-1],
               "re": res.trace.re[-1], "normest": res.trace.normest, "condest": res.trace.condest}}
print(json.dumps(out), flush=True)
t0 = time.time()
a_h = np.empty((m, n))
blk = 250_000
for i in range(0, m, blk):
    a_h[i:i + blk] = p.a[i:i + blk].cpu().numpy()
b_h = p.b.cpu().numpy()
r_h = p.truth.r.cpu().numpy()
x_true = p.truth.x
del p
torch.cuda.empty_cache()
out["d2h_s"] = time.time() - t0
t0 = time.time()
x_ref, tr_ref = orc.iterative_sketching(a_h, b_h, orc.Config(d=d, variant=variant, rng_seed=seed),
                                        orc.Truth(x=x_true, r=r_h, kappa=kappa, beta=beta))
out["oracle_solve_s"] = time.time() - t0
dev_x = float(np.linalg.norm(res.solution - x_ref) / np.linalg.norm(x_ref))
out["oracle"] = {"iterations": len(tr_ref.iterates) - 1, "stop": tr_ref.stop_reason, "fe": tr_ref.fe[-1],
                 "re": tr_ref.re[-1], "normest": tr_ref.normest, "condest": tr_ref.condest}
out["x_dev_rel"] = dev_x
out["bound_10kappa_u_plus_fe_ref"] = 10 * kappa * U + tr_ref.fe[-1]
out["checks"] = {"fe_within_2x": res.trace.fe[-1] <= 2 * tr_ref.fe[-1],
                 "re_within_2x": res.trace.re[-1] <= 2 * tr_ref.re[-1],
                 "stated_bound": dev_x <= out["bound_10kappa_u_plus_fe_ref"],
                 "same_stop": res.trace.stop_reason == tr_ref.stop_reason}
print(json.dumps(out), flush=True)
os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
with open(os.path.join(ROOT, "gpurun_out" if os.path.isdir(os.path.join(ROOT, "gpurun_out")) else "profiles",
                       f"c4_parity_{variant}_s{seed}.json"), "w") as f:
    json.dump(out, f, indent=1)

"""Per-phase device timing of one C2 solve (CUDA events, synchronised)."""
import ctypes, sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2311_04362_b200 as itsk
from paper_2311_04362_b200 import _lib, solvers
from paper_2311_04362_b200 import device as dv
from paper_2311_04362_b200.embed import pcg_state
from paper_2311_04362_b200.linalg import start_vector, normest_steps

cfgname = sys.argv[1] if len(sys.argv) > 1 else "c2"
variant = sys.argv[2] if len(sys.argv) > 2 else "basic"
gen = sys.argv[3] if len(sys.argv) > 3 else None
from bench import CONFIGS, make_problem
m, n, kappa, beta, d, zeta = CONFIGS[cfgname]
t0 = time.perf_counter()
p, _, _ = make_problem(cfgname, 0)
torch.cuda.synchronize()
print(f"generate {time.perf_counter() - t0:.1f} s", flush=True)
dev = torch.device("cuda")
lib = _lib.lib_for_device(0)
at = p.a if isinstance(p.a, torch.Tensor) else torch.from_numpy(p.a).to(dev)
bt = p.b if isinstance(p.b, torch.Tensor) else torch.from_numpy(p.b).to(dev)
cfg = itsk.SolverConfig(d=d, zeta=zeta, variant=variant)
for _ in range(3):
    res = itsk.iterative_sketching(at, bt, cfg, residuals="last")
ws = next(iter(solvers._WS.values()))
st = torch.cuda.current_stream(); s = int(st.cuda_stream)
def T(fn, reps=5):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize(); e0 = torch.cuda.Event(True); e1 = torch.cuda.Event(True)
        w0 = time.perf_counter(); e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append((e0.elapsed_time(e1), 1e3*(time.perf_counter()-w0)))
    return np.median([t[0] for t in ts]), np.median([t[1] for t in ts])
words, h, pend = pcg_state(0)
out = {}
out["pattern"] = T(lambda: _lib.check(lib.itsk_sparse_sign_pattern(d, m, zeta, words, h, pend, dv.ptr(ws.rows), dv.ptr(ws.neg), dv.ptr(ws.sk_ptr), dv.ptr(ws.sk_src), dv.ptr(ws.pat_ws), ws.pat_ws.numel(), s)))
out["sketch"] = T(lambda: _lib.check(lib.itsk_sketch(dv.ptr(at), m, n, n, dv.ptr(bt), dv.ptr(ws.sk_ptr), dv.ptr(ws.sk_src), d, zeta, dv.ptr(ws.W), ws.ldw, s)))
W0 = ws.W.clone()
def qr():
    ws.W.copy_(W0)
    _lib.check(lib.itsk_qr_aug(dv.ptr(ws.W), d, n, ws.ldw, dv.ptr(ws.R), dv.ptr(ws.z), dv.ptr(ws.qr_ws), ws.qr_ws.numel(), s))
out["qr(+copy)"] = T(qr)
out["copyW"] = T(lambda: ws.W.copy_(W0))
out["trsv_x0"] = T(lambda: _lib.check(lib.itsk_trsv(dv.ptr(ws.R), n, dv.ptr(ws.z), dv.ptr(ws.xs[0]), 0, s)))
out["trsv_rp_x0"] = T(lambda: _lib.check(lib.itsk_trsv_rp(dv.ptr(ws.R), dv.ptr(ws.Rp), n, dv.ptr(ws.z), dv.ptr(ws.xs[0]), 0, s)))
out["normest"] = T(lambda: _lib.check(lib.itsk_normest(dv.ptr(ws.R), n, dv.ptr(ws.v0), normest_steps(n), dv.ptr(ws.est), None, s)))
out["condest"] = T(lambda: _lib.check(lib.itsk_condest(dv.ptr(ws.R), n, dv.ptr(ws.v0), dv.ptr(ws.est)+8, None, s)))
cond_ws = torch.empty(n * n, dtype=torch.float64, device=dev)
out["condest_ws"] = T(lambda: _lib.check(lib.itsk_condest_ws(dv.ptr(ws.R), n, dv.ptr(ws.v0), dv.ptr(ws.est)+8, dv.ptr(ws.Rp), dv.ptr(cond_ws), cond_ws.numel(), s)))
out["condest_Rp"] = T(lambda: _lib.check(lib.itsk_condest(dv.ptr(ws.R), n, dv.ptr(ws.v0), dv.ptr(ws.est)+8, dv.ptr(ws.Rp), s)))
out["normest_Rp"] = T(lambda: _lib.check(lib.itsk_normest(dv.ptr(ws.R), n, dv.ptr(ws.v0), normest_steps(n), dv.ptr(ws.est), dv.ptr(ws.Rp), s)))
p_ = solvers._loop_params(ws, at, n, cfg, 1.0, 0.0, None)
p_.b = dv.ptr(bt)  # the solver reads a device b in place (ws.b is not filled)
def loop():
    solvers.run_loop(lib, ws, p_, True, s)
out["loop(graph)"] = T(loop)
out["loop(steps)"] = T(lambda: solvers.run_loop(lib, ws, p_, False, s))
out["trsv_pair"] = T(lambda: _lib.check(lib.itsk_trsv_pair(dv.ptr(ws.R), n, dv.ptr(ws.cs), dv.ptr(ws.z), None, s)))
out["full_solve"] = T(lambda: itsk.iterative_sketching(at, bt, cfg, residuals="last"))
# residuals="all": normest / condest deferred beside the loop's first iterations
out["full_solve_all"] = T(lambda: itsk.iterative_sketching(at, bt, cfg, residuals="all"))
res = itsk.iterative_sketching(at, bt, cfg, p.truth, residuals="last")
print(f"{cfgname} {variant} iters={res.iterations} stop={res.trace.stop_reason} "
      f"fe={res.trace.fe[-1]:.3e} re={res.trace.re[-1]:.3e} normest={res.trace.normest:.4e} condest={res.trace.condest:.4e}")
for k, (g, w) in out.items():
    print(f"{k:14s} device {g:9.3f} ms   wall {w:9.3f} ms")

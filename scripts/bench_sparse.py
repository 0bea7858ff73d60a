"""Sparse-A benchmark (§3.5 regime): gen_sparse
(3 nonzeros +-1 per row, Gaussian b), d = 30n, zeta = 8, basic, max_iters
fixed (the stopping rule does not fire on these inconsistent systems — the
reference's own sparsebench runs to max_iters too).

    python scripts/bench_sparse.py [--m 3000000] [--n 1000] [--iters 20] [--steps 5] [--warmup 3]

Prints one JSON line:
  value     solve time, CSR (and its CSC plan) resident in HBM (CUDA events)
  e2e       the same solve from the scipy CSR on the host: upload + plan
            (CSC copy) + solve + trace readback inside the timed region
  roofline  the sparse pass (k_csr_rows + k_csc_chunks + k_csr_finish):
            algorithmic bytes 24 nnz + 8 (m+1) + 24 m per pass (CSR and CSC
            entries, row pointers, b / r_prev / r) over its event-timed launch
  cpu_baseline  the oracle (the reference's scipy calls) on the same instance
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=3_000_000)
    ap.add_argument("--n", type=int, default=1000)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    import torch

    import paper_2311_04362_b200 as itsk
    from bench import ClockSampler, blas_threads, peaks
    from paper_2311_04362_b200 import _lib

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    lib = _lib.lib_for_device(0)
    m, n = args.m, args.n
    d = 30 * n
    prob = itsk.gen_sparse(m, n, 0)
    nnz = prob.a.nnz
    cfg = itsk.SolverConfig(d=d, zeta=8, max_iters=args.iters, rng_seed=0)
    A = itsk.CsrMatrix.from_scipy(prob.a, dev)
    b_dev = torch.from_numpy(prob.b).to(dev)
    stream = torch.cuda.current_stream(dev)

    def timed(fn, steps):
        ts, res = [], None
        for _ in range(steps):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            res = fn()
            e1.record(stream)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        return ts, res

    solve_dev = lambda: itsk.iterative_sketching(A, b_dev, cfg, residuals="last")  # noqa: E731
    solve_host = lambda: itsk.iterative_sketching(prob.a, prob.b, cfg, residuals="last")  # noqa: E731
    for _ in range(args.warmup):
        solve_dev()
    l0 = lib.itsk_launch_count()
    with ClockSampler(0) as clk:
        t_dev, res = timed(solve_dev, args.steps)
    l1 = lib.itsk_launch_count()
    for _ in range(1):
        solve_host()
    t_e2e, _ = timed(solve_host, args.steps)
    # the pass alone
    x = torch.from_numpy(res.solution).to(dev)
    r_prev = torch.zeros(m, dtype=torch.float64, device=dev)
    r_out = torch.empty(m, dtype=torch.float64, device=dev)
    for _ in range(3):
        A.pass_(b_dev, x, r_out=r_out, r_prev=r_prev)
    reps = 30
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        A.pass_(b_dev, x, r_out=r_out, r_prev=r_prev)
    e1.record(stream)
    torch.cuda.synchronize()
    pass_ms = e0.elapsed_time(e1) / reps
    alg = 24.0 * nnz + 8.0 * (m + 1) + 24.0 * m
    peak, kind = peaks()
    achieved = alg / (pass_ms * 1e-3) / 1e9
    out = {
        "metric": "sparse fp64 LS solve time (PAPER §3.5 regime) & sparse pass HBM GB/s",
        "value": statistics.median(t_dev), "unit": "ms", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "higher_is_better": False, "dtype": "f64", "data": "synthetic (gen_sparse, seed 0)",
        "config": {"workload": f"sparse: iterative_sketching gen_sparse m={m} n={n} nnz={nnz} d={d} zeta=8 "
                               f"variant=basic max_iters={args.iters}",
                   "l2": f"CSR+CSC {(24 * nnz + 8 * m) / 2**20:.0f} MiB > L2 (126 MB)"},
        "e2e": {"value": statistics.median(t_e2e), "unit": "ms",
                "h2d_bytes_per_step": int(20 * nnz + 8 * (m + 1) + 8 * m),
                "d2h_bytes_per_step": int(8 * ((args.iters + 1) * n + 4 * (args.iters + 1) + 2) + 48)},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "peak_kind": kind, "traffic": None,
                     "kernel": "k_csr_rows + k_csc_chunks + k_csr_finish (r = b - Ax bitwise, c = A'r)",
                     "bytes_per_launch": alg, "ms_per_launch": pass_ms},
        "gpu_launches": int((l1 - l0) + args.steps * 4 * res.iterations),
        "iterations": res.iterations, "stop_reason": res.trace.stop_reason,
        "clocks": clk.summary(),
    }
    if not args.no_cpu_baseline:
        from oracle import itsketch_oracle as orc

        t0 = time.perf_counter()
        xo, tro = orc.iterative_sketching(prob.a, prob.b, orc.Config(d=d, zeta=8, max_iters=args.iters))
        cpu_ms = 1e3 * (time.perf_counter() - t0)
        out["cpu_baseline"] = {"value": cpu_ms, "unit": "ms", "cores": blas_threads(), "kind": "port",
                               "sample": "1 full solve on the oracle (the reference's scipy sparse calls; "
                                         "scipy's sparse products are single-threaded)"}
        out["x_rel_diff_vs_oracle"] = float(np.linalg.norm(res.solution - xo) / np.linalg.norm(xo))
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()

"""Benchmark: fp64 iterative-sketching LS solve on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--config c2] [--variant basic|damped|momentum]

One "step" = one full `iterative_sketching` solve of the BASELINE workload
(configs[1], "C2": gen_randsvd(200000, 200, kappa=1e10, beta=1e-12, seed=0),
d = 20n = 4000, zeta = 8, reference-default basic variant, max_iters = 50):
device pattern -> S·[A|b] -> QR -> x0 -> normest/condest -> refinement loop
-> trace readback.

  value   solve time (ms) with A, b resident in HBM (CUDA events, max over ranks)
  e2e     same solve through the public API from pinned host numpy arrays:
          H2D of A and b plus the D2H of solution/trace inside the timed region
  roofline  the fused r=b-Ax / c=A'r pass (the loop's dominant kernel), timed
          with CUDA events on its own stream: 8*m*n algorithmic bytes / launch
  cpu_baseline  the CPU oracle (numpy/OpenBLAS restatement of the reference)
          on the same instance, all host cores

--impl reference: the reference's CPU implementation of the path (the oracle
port — the reference is pure Python and cannot travel to the GPU box) timed on
the host on the same config; rank 0 only.
A (320 MB) is larger than the 126 MB L2, so every pass streams from HBM.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fp64 LS solve time & fused Aᵀ(b−Ax) HBM GB/s (% of peak) at 1/2/4/8 B200"

CONFIGS = {
    # name: (m, n, kappa, beta, d, zeta)
    "c1": (4000, 50, 1e10, 1e-6, 1000, 8),
    "c2": (200000, 200, 1e10, 1e-12, 4000, 8),
    "c3": (1000000, 500, 1e15, 1e-3, 10000, 8),
    "c4": (4000000, 2000, 1e8, 1e-6, 24000, 8),
}
# host numpy generator (the reference's construction and draw order) where it
# is feasible; the device generator (instances.gen_randsvd_device) for C4
GEN = {"c1": "host", "c2": "host", "c3": "host", "c4": "device"}
# C4: d = 12n puts basic outside its contraction margin; the
# headline is momentum
DEFAULT_VARIANT = {"c4": "momentum"}
# configs whose oracle solve is too long for a bench run: phase-sampled estimate
SAMPLED = {"c4"}
# iteration count used by the sampled estimate when the reference arm runs
# alone (the GPU arm uses its own count); C4 momentum: measured on the GPU
REF_ITERS = {"c4": 18}


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """SM clock + throttle reasons sampled through NVML every 5 ms while the
    timed region runs (nvidia-smi's 100 ms floor would see ~1 sample of a
    60 ms region)."""

    def __init__(self, index: int, period_s: float = 0.005):
        self.index = index
        self.period = period_s
        self.samples: list[tuple[float, int]] = []
        self.smax = None
        self._stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.smax = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self.thread = threading.Thread(target=self._run, daemon=True)
            self.thread.start()
        except Exception:
            self._nv = None
        return self

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                clk = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
                rsn = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                self.samples.append((float(clk), int(rsn)))
            except Exception:
                pass
            time.sleep(self.period)

    def __exit__(self, *exc):
        self._stop.set()
        if getattr(self, "thread", None) is not None:
            self.thread.join(timeout=2)

    def summary(self):
        names = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
                 0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown"}
        reasons = set()
        for _, r in self.samples:
            for bit, nm in names.items():
                if r & bit:
                    reasons.add(nm)
        sm = [c for c, _ in self.samples]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.smax,
                "reasons": sorted(reasons), "samples": len(sm), "source": "nvml, 5 ms"}


def make_problem(name: str, seed: int = 0, gen: str | None = None):
    m, n, kappa, beta, d, zeta = CONFIGS[name]
    if (gen or GEN[name]) == "device":
        from paper_2311_04362_b200.instances import gen_randsvd_device

        return gen_randsvd_device(m, n, kappa, beta, seed), d, zeta
    from paper_2311_04362_b200 import gen_randsvd

    return gen_randsvd(m, n, kappa, beta, seed), d, zeta


def host_ram_bytes() -> int:
    try:
        import psutil

        return int(psutil.virtual_memory().available)
    except Exception:
        return 0


def cpu_solve_time(a, b, d, zeta, variant, reps):
    from oracle import itsketch_oracle as orc

    times = []
    res = None
    for _ in range(reps):
        t0 = time.perf_counter()
        res = orc.iterative_sketching(a, b, orc.Config(d=d, zeta=zeta, variant=variant))
        times.append(time.perf_counter() - t0)
    return times, res


SAMPLE_ROWS = 250_000


def cpu_sampled_estimate(a_s, b_s, m, d, zeta, iters, seed=0):
    """Oracle solve time at a size too large to run whole in minutes: the
    reference's phases timed on a bounded sample and scaled to the full size.
      pattern + S·[A|b]   on the first SAMPLE_ROWS rows, x m/SAMPLE_ROWS
      QR                  of a d x (n+1) matrix (the sketch's shape), once
      refinement pass     r = b - A x, c = A'r on the sample, x m/SAMPLE_ROWS,
                          times (iters + 1) passes (+ two n x n solves each)
    Returns (ms, description)."""
    from oracle import itsketch_oracle as orc

    ms, n = (int(v) for v in a_s.shape)
    scale = m / ms
    t0 = time.perf_counter()
    pat = orc.sparse_sign_pattern(d, ms, zeta, seed)
    orc.sketch_apply(pat, np.column_stack([a_s, b_s]))
    t_sketch = (time.perf_counter() - t0) * scale
    w = np.random.default_rng(1).standard_normal((d, n + 1))
    t0 = time.perf_counter()
    q, r = orc.householder_qr_econ(w[:, :n])
    t_qr = time.perf_counter() - t0
    x = np.random.default_rng(2).standard_normal(n)
    reps = 3
    t0 = time.perf_counter()
    for _ in range(reps):
        res = b_s - a_s @ x
        c = a_s.T @ res
    t_pass = (time.perf_counter() - t0) / reps * scale
    t0 = time.perf_counter()
    for _ in range(reps):
        orc.tri_solve_upper(r, orc.tri_solve_upper_transpose(r, c))
    t_tri = (time.perf_counter() - t0) / reps
    total = t_sketch + t_qr + (iters + 1) * t_pass + iters * t_tri
    desc = (f"extrapolated: oracle pattern+sketch and one r=b-Ax, c=A'r pass on the first {ms} of {m} rows "
            f"(x{scale:.1f}), QR of a {d}x{n} matrix, trisolve pair; {iters} iterations "
            f"[sketch {t_sketch:.2f} s, qr {t_qr:.2f} s, pass {t_pass:.3f} s, tri {t_tri:.4f} s]")
    return 1e3 * total, desc


def blas_threads():
    try:
        from threadpoolctl import threadpool_info

        return max((i.get("num_threads", 1) for i in threadpool_info()), default=os.cpu_count())
    except Exception:
        return os.cpu_count()


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    if args.config in SAMPLED:
        return run_reference_sampled(args)
    prob, d, zeta = make_problem(args.config)
    m, n = prob.a.shape
    _, _ = cpu_solve_time(prob.a, prob.b, d, zeta, args.variant, args.warmup)
    times, res = cpu_solve_time(prob.a, prob.b, d, zeta, args.variant, args.steps)
    ms = 1e3 * statistics.median(times)
    cores = blas_threads()
    line = {
        "impl": "reference", "metric": METRIC, "value": ms, "unit": "ms", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (gen_randsvd, seed 0)",
        "config": {"workload": f"{args.config}: iterative_sketching m={m} n={n} d={d} zeta={zeta} "
                               f"variant={args.variant}", "parallelism": "host threads (OpenBLAS)"},
        "cpu_baseline": {"value": ms, "unit": "ms", "cores": cores, "kind": "port",
                         "sample": f"{args.steps} full solves of {args.config} on the oracle "
                                   "(numpy/scipy restatement of itsketch.iterative_sketching)"},
        "e2e": {"value": ms, "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "iterations": len(res[1].iterates) - 1, "stop_reason": res[1].stop_reason,
    }
    print(json.dumps(line), flush=True)
    return 0


def run_reference_sampled(args):
    """--impl reference for a config whose oracle solve does not fit a bench
    run: each step is the phase-sampled estimate (cpu_sampled_estimate) on a
    Gaussian row block of the config's shape (the oracle's phase times do not
    depend on the values)."""
    m, n, kappa, beta, d, zeta = CONFIGS[args.config]
    rng = np.random.default_rng(0)
    ms = min(m, SAMPLE_ROWS)
    a_s = rng.standard_normal((ms, n))
    b_s = rng.standard_normal(ms)
    iters = REF_ITERS[args.config]
    for _ in range(args.warmup):
        cpu_sampled_estimate(a_s[:2000, :50], b_s[:2000], 2000, 200, zeta, 1)
    vals, desc = [], ""
    for _ in range(args.steps):
        v, desc = cpu_sampled_estimate(a_s, b_s, m, d, zeta, iters)
        vals.append(v)
    ms_val = statistics.median(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": ms_val, "unit": "ms", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_val, "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (Gaussian row sample)",
        "config": {"workload": f"{args.config}: iterative_sketching m={m} n={n} d={d} zeta={zeta} "
                               f"variant={args.variant}", "parallelism": "host threads (OpenBLAS)"},
        "cpu_baseline": {"value": ms_val, "unit": "ms", "cores": blas_threads(), "kind": "port", "sample": desc},
        "e2e": {"value": ms_val, "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "iterations": iters,
    }
    print(json.dumps(line), flush=True)
    return 0


def fused_pass_timing(lib, at, bt, x, n_launch=30):
    """Average device time of the fused pass (CUDA events on its stream)."""
    import ctypes

    import torch

    from paper_2311_04362_b200 import _lib
    from paper_2311_04362_b200 import device as dv

    m, n = at.shape
    dev = at.device
    nb = ctypes.c_int64()
    _lib.check(lib.itsk_pass_workspace(m, n, ctypes.byref(nb)))
    ws = dv.workspace(nb.value, dev)
    r_prev = torch.zeros(m, dtype=torch.float64, device=dev)
    r_out = torch.empty(m, dtype=torch.float64, device=dev)
    cs = torch.empty(n + 8, dtype=torch.float64, device=dev)
    stream = torch.cuda.Stream(dev)
    with torch.cuda.stream(stream):
        sp = int(stream.cuda_stream)
        _lib.check(lib.itsk_pass_workspace_init(dv.ptr(ws), m, n, sp))

        def launch():
            _lib.check(lib.itsk_fused_pass_ex(dv.ptr(at), m, n, int(at.stride(0)), dv.ptr(bt), 1.0, dv.ptr(x),
                                              dv.ptr(r_prev), dv.ptr(r_out), None, dv.ptr(cs), dv.ptr(ws),
                                              ws.numel(), _lib.PASS_WS_READY, sp))

        for _ in range(5):
            launch()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        stream.synchronize()
        e0.record(stream)
        for _ in range(n_launch):
            launch()
        e1.record(stream)
        stream.synchronize()
    return e0.elapsed_time(e1) / n_launch  # ms per launch (pass + finalize)


def run_b200(args):
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # --sharded: the row-sharded path even at N = 1 (checks the N > 1 code
    # path on one GPU; needs the torchrun environment)
    dist_on = world > 1 or args.sharded
    if dist_on:
        import torch.distributed as tdist

        tdist.init_process_group("nccl", device_id=dev)

    import paper_2311_04362_b200 as itsk
    from paper_2311_04362_b200 import _lib
    from paper_2311_04362_b200.dist import iterative_sketching_sharded, shard_bounds

    lib = _lib.lib_for_device(local)
    prob, d, zeta = make_problem(args.config)
    m, n = prob.a.shape
    cfg = itsk.SolverConfig(d=d, zeta=zeta, variant=args.variant)
    r0, r1 = shard_bounds(m, world, rank)
    on_device = isinstance(prob.a, torch.Tensor)
    a_bytes = 8 * (r1 - r0) * n
    # pinned host copies (e2e input) and HBM-resident copies (value input)
    do_e2e = not on_device or host_ram_bytes() > 2 * a_bytes + (8 << 30)
    a_pin = b_pin = None
    if on_device:
        a_dev = prob.a[r0:r1]
        b_dev = prob.b[r0:r1].contiguous()
        x_true = prob.truth.x
        if do_e2e:
            a_pin = torch.empty(tuple(a_dev.shape), dtype=torch.float64, pin_memory=True)
            a_pin.copy_(a_dev)
            b_pin = b_dev.cpu().pin_memory()
    else:
        a_pin = torch.empty((r1 - r0, n), dtype=torch.float64, pin_memory=True)
        a_pin.copy_(torch.from_numpy(np.ascontiguousarray(prob.a[r0:r1])))
        b_pin = torch.empty(r1 - r0, dtype=torch.float64, pin_memory=True)
        b_pin.copy_(torch.from_numpy(np.ascontiguousarray(prob.b[r0:r1])))
        a_dev = a_pin.to(dev)
        b_dev = b_pin.to(dev)
        x_true = prob.truth.x
    torch.cuda.synchronize()

    def solve(a_in, b_in):
        if dist_on:
            return iterative_sketching_sharded(a_in, b_in, cfg, m, r0, residuals="all")
        # the reference keeps every residual (solvers.py:245-246); that also lets
        # normest / condest run beside the first iterations (deferred estimates)
        return itsk.iterative_sketching(a_in, b_in, cfg, residuals="all")

    def barrier():
        if dist_on:
            tdist.barrier()
        torch.cuda.synchronize()

    def timed(a_in, b_in, steps):
        stream = torch.cuda.current_stream(dev)
        times = []
        res = None
        for _ in range(steps):
            barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            res = solve(a_in, b_in)
            e1.record(stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
        return times, res

    for _ in range(args.warmup):
        solve(a_dev, b_dev)
    barrier()
    l0 = lib.itsk_launch_count()
    with ClockSampler(local) as clk:
        t_dev, res = timed(a_dev, b_dev, args.steps)
    l1 = lib.itsk_launch_count()
    t_e2e = [float("nan")]
    if do_e2e:
        for _ in range(min(args.warmup, 1 if on_device else args.warmup)):
            solve(a_pin.numpy(), b_pin.numpy())
        t_e2e, res_e2e = timed(a_pin.numpy(), b_pin.numpy(), args.steps)
    iters = res.iterations
    # graph-body kernels (fused pass, tail) run once per iteration
    # (the sharded loop is one graph too when the peer exchange carries its sums)
    graph_loop = (not dist_on) or bool(getattr(res, "peer_exchange", False))
    launches = (l1 - l0) + args.steps * 2 * iters if graph_loop else (l1 - l0)

    def reduce_max(v):
        if not dist_on:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        return float(t.item())

    ms_dev = reduce_max(statistics.median(t_dev))
    ms_e2e = reduce_max(statistics.median(t_e2e)) if do_e2e else None
    x_dev = torch.from_numpy(res.solution).to(dev)
    pass_ms = reduce_max(fused_pass_timing(lib, a_dev, b_dev, x_dev))
    peak, peak_kind = peaks()
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "pass_traffic.json")) as f:
            tr = json.load(f)
        if tr.get("m") == r1 - r0 and tr.get("n") == n:
            traffic = tr["dram_bytes_per_launch"]
    except Exception:
        pass
    alg_bytes = 8.0 * (r1 - r0) * n
    achieved = alg_bytes / (pass_ms * 1e-3) / 1e9
    out = None
    if rank == 0:
        fe = float(np.linalg.norm(res.solution - x_true) / np.linalg.norm(x_true))
        out = {
            "metric": METRIC, "value": ms_dev, "unit": "ms", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_dev, "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (gen_randsvd, seed 0; no dataset)",
            "config": {"workload": f"{args.config}: iterative_sketching m={m} n={n} d={d} zeta={zeta} "
                                   f"variant={args.variant} max_iters={cfg.max_iters}",
                       "global_rows": m, "cols": n, "parallelism": f"row-shard x{world}",
                       "loop_exchange": (None if not dist_on else
                                         "peer memory (pass stores to every rank, tail sums; one CUDA graph)"
                                         if graph_loop else "nccl allreduce per iteration"),
                       "generator": GEN[args.config],
                       "l2": f"A ({a_bytes / 2**20:.0f} MiB per GPU) > L2 (126 MB): every pass streams from HBM, "
                             "no flush needed"},
            "e2e": ({"value": ms_e2e, "unit": "ms", "h2d_bytes_per_step": int(8 * m * n + 8 * m),
                     "d2h_bytes_per_step": int(8 * ((cfg.max_iters + 1) * n + 4 * (cfg.max_iters + 1) + 2) + 48)}
                    if do_e2e else {"value": None, "unit": "ms",
                                    "skipped": "host RAM below 2x A for the pinned copy"}),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "peak_kind": peak_kind, "traffic": traffic,
                         "kernel": "k_pass_tma (fused r=b-Ax, c=A'r, norms, in-kernel partial reduction)",
                         "bytes_per_launch": alg_bytes, "ms_per_launch": pass_ms},
            "gpu_launches": int(launches),
            "iterations": iters, "stop_reason": res.trace.stop_reason, "fe": fe,
            "passes_per_solve": iters + 1,
            "clocks": clk.summary(),
        }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        if args.config not in SAMPLED:
            times, ores = cpu_solve_time(prob.a, prob.b, d, zeta, args.variant, 1)
            cpu_ms, sample = 1e3 * times[0], f"1 full solve of {args.config} on the oracle (numpy/OpenBLAS)"
        else:
            ms_rows = min(m, SAMPLE_ROWS)
            a_s, b_s = prob.a[:ms_rows], prob.b[:ms_rows]
            if isinstance(a_s, torch.Tensor):
                a_s, b_s = a_s.cpu().numpy(), b_s.cpu().numpy()
            cpu_ms, sample = cpu_sampled_estimate(a_s, b_s, m, d, zeta, iters)
        out["cpu_baseline"] = {"value": cpu_ms, "unit": "ms", "cores": blas_threads(), "kind": "port",
                               "sample": sample}
    if rank == 0:
        print(json.dumps(out), flush=True)
    if dist_on:
        tdist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--variant", default=None, choices=["basic", "damped", "momentum"])
    ap.add_argument("--sharded", action="store_true",
                    help="run the row-sharded (multi-GPU) path even with one rank (under torchrun)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.variant is None:
        args.variant = DEFAULT_VARIANT.get(args.config, "basic")
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())

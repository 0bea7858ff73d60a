"""Experiment CLI with a device flag.

Mirrors the reference's runner (/root/reference/pkg/src/itsketch/cli.py):
the same subcommand names, flags, CSV files (`# schema=v1` line, header,
rows sorted by their string form, floats written with repr — cli.py:38,58-64)
and exit codes (0 ok, 1 solver divergence, 2 I/O error, 64 bad flags —
cli.py:41-44).  Every solve runs on the B200 path; `--device cuda[:K]` picks
the GPU.  Subcommands on the north-star path:

  solve        cli.py:102-123   one generated instance -> x CSV + summary CSV
  convergence  cli.py:126-160   per-iteration traces + Householder-QR row
  compare      cli.py:179-190   IS basic/damped/momentum vs sketch-and-precondition
  dims         cli.py:193-199   embedding-dimension table (host arithmetic)
  sparsebench  cli.py:259-274   sparse +-1 instances (gen_sparse), timing scan

`bad` (the deliberately unstable baselines) and `kernel` (kernel-regression
data) are outside this repository's scope: argparse rejects
them with exit code 64 like any unknown subcommand.

Run as `python -m paper_2311_04362_b200 <subcommand> ...`.
"""

from __future__ import annotations

import argparse
import math
import sys
import time

import numpy as np

SCHEMA_LINE = "# schema=v1"

EXIT_OK = 0
EXIT_DIVERGED = 1
EXIT_IO = 2
EXIT_USAGE = 64

TRACE_HEADER = "method,kappa,resnorm,iter,fe,re,be,res_change,bound_fe,bound_re"


class _Parser(argparse.ArgumentParser):
    """argparse exits 2 on bad flags; the reference's contract is 64 (cli.py:47-50)."""

    def error(self, message: str) -> None:
        self.print_usage(sys.stderr)
        self.exit(EXIT_USAGE, f"{self.prog}: error: {message}\n")


# --------------------------------------------------------------------------
# CSV output (cli.py:58-64, problems.py:177-186)
# --------------------------------------------------------------------------
def _fmt(v) -> str:
    return repr(v) if isinstance(v, float) else str(v)


def write_table(path: str, header: str, rows: list[list]) -> None:
    """`# schema=v1`, the header, then the rows ordered by their string form."""
    rows = sorted(rows, key=lambda row: [str(v) for v in row])
    with open(path, "w") as f:
        f.write(SCHEMA_LINE + "\n")
        f.write(header + "\n")
        for row in rows:
            f.write(",".join(_fmt(v) for v in row) + "\n")


def save_numeric_csv(path: str, header: list[str], values: np.ndarray) -> None:
    """Numeric CSV with shortest round-trip decimals (problems.py:177-186)."""
    with open(path, "w", newline="") as f:
        f.write(",".join(header) + "\r\n")
        for row in np.atleast_2d(values):
            f.write(",".join(repr(float(v)) for v in row) + "\r\n")


# --------------------------------------------------------------------------
# Host-side formulas the CLI needs (not on the solve path)
# --------------------------------------------------------------------------
class RateHypothesisError(ValueError):
    """A bound was requested outside the epsilon range its theorem covers."""


def _check_eps(eps: float, lo_open: bool = False) -> None:
    ok = (0 < eps < 1) if lo_open else (0 <= eps < 1)
    if not ok:
        raise RateHypothesisError(f"need {'0 <' if lo_open else '0 <='} eps < 1, got {eps}")


def bound_curve(variant: str, eps: float, kappa: float, norm_a: float, norm_r: float, iters: int,
                first_iter: int = 0) -> tuple[np.ndarray, np.ndarray]:
    """Exact-arithmetic error bounds of the paper's convergence theorems
    (Thm. 3 / 5 / 6; the reference's theoretical_bound_curve,
    solvers.py:140-171): RE_i <= C(eps) g(eps)^i ||r||, FE_i = RE_i kappa/||A||.
    basic: g = (2-e)e/(1-e)^2, C = (8-2 sqrt 2) sqrt e (needs e < 1-1/sqrt 2);
    damped: g = 2e/(1+e^2), C = 2(1+e) sqrt e/(1-e)^2;
    momentum: g = e, C = 8 sqrt 2 (1+e)/((1-e)^2 sqrt e) times (i-1), i >= 2."""
    i = np.arange(first_iter, iters + 1, dtype=float)
    e = float(eps)
    if variant == "basic":
        if not 0 <= e < 1 - 1 / math.sqrt(2):
            raise RateHypothesisError(f"basic bound needs eps < 1 - 1/sqrt(2), got {e}")
        g = (2 - e) * e / (1 - e) ** 2
        re = (8 - 2 * math.sqrt(2)) * math.sqrt(e) * g ** i * norm_r
    elif variant == "damped":
        _check_eps(e)
        re = 2 * (1 + e) * math.sqrt(e) / (1 - e) ** 2 * (2 * e / (1 + e * e)) ** i * norm_r
    elif variant == "momentum":
        _check_eps(e, lo_open=True)
        if first_iter < 2:
            raise RateHypothesisError("momentum bound is stated for i >= 2")
        re = 8 * math.sqrt(2) * (1 + e) / ((1 - e) ** 2 * math.sqrt(e)) * (i - 1) * e ** i * norm_r
    else:
        raise ValueError(f"unknown variant {variant!r}")
    return re * (kappa / norm_a), re


def choose_dim(m: int, n: int, accuracy_u: float, variant: str = "basic") -> int:
    """Embedding dimension of the paper's cost balance (embed.py:138-158):
    basic d = max(20n, ceil((6+4 sqrt 2) n exp W((6-4 sqrt 2) m/n^2 log(1/u))));
    damped / momentum d = max(4n, ceil(a n exp W(4m/(a n^2) log(1/u)))), a = 2 / 1."""
    from scipy.special import lambertw

    if m < n or n < 1:
        raise ValueError(f"need m >= n >= 1, got m={m}, n={n}")
    if not 0 < accuracy_u < 1:
        raise ValueError(f"accuracy must be in (0, 1), got {accuracy_u}")
    log_inv_u = math.log(1.0 / accuracy_u)

    def w0(x: float) -> float:
        if x < -1 / math.e:
            raise ValueError("lambert_w0 needs x >= -1/e")
        return float(lambertw(x, 0).real)

    if variant == "basic":
        arg = (6 - 4 * math.sqrt(2)) * (m / n ** 2) * log_inv_u
        return max(math.ceil((6 + 4 * math.sqrt(2)) * n * math.exp(w0(arg))), 20 * n)
    if variant in ("damped", "momentum"):
        a = 2.0 if variant == "damped" else 1.0
        arg = (4 * m / (a * n ** 2)) * log_inv_u
        return max(math.ceil(a * n * math.exp(w0(arg))), 4 * n)
    raise ValueError(f"unknown variant {variant!r}")


# --------------------------------------------------------------------------
# Subcommands
# --------------------------------------------------------------------------
def _select_device(spec: str):
    import torch

    if not spec.startswith("cuda"):
        raise SystemExit(f"error: --device must be cuda or cuda:K (there is no CPU path), got {spec!r}")
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2311_04362_b200 needs a CUDA (sm_100) device; there is no CPU path")
    dev = torch.device(spec)
    torch.cuda.set_device(dev.index if dev.index is not None else 0)
    return dev


def _resolve_d(args, m: int, n: int, variant: str) -> int:
    if args.d == "auto":
        return choose_dim(m, n, args.accuracy, variant)
    return int(args.d)


def _solver_cfg(args, m: int, n: int, variant: str | None = None, seed: int | None = None,
                init: str = "sketch_and_solve"):
    from .solvers import SolverConfig

    variant = variant or args.variant
    return SolverConfig(d=_resolve_d(args, m, n, variant), zeta=args.zeta, variant=variant, init=init,
                        max_iters=args.max_iters, rng_seed=args.seed[0] if seed is None else seed,
                        track_be=(args.metrics == "full"))


def _last(v):
    return float(v[-1]) if v else float("nan")


def _trace_rows(method: str, kappa: float, beta: float, res, bounds=None) -> list[list]:
    t = res.trace
    rows = []
    for i in range(len(t.iterates)):
        fe = float(t.fe[i]) if t.fe else float("nan")
        re = float(t.re[i]) if t.re else float("nan")
        be = float(t.be[i]) if i < len(t.be) else float("nan")
        chg = float(t.residual_changes[i - 1]) if i >= 1 else float("nan")
        bf, br = float("nan"), float("nan")
        if bounds is not None and i < len(bounds[0]):
            bf, br = float(bounds[0][i]), float(bounds[1][i])
        rows.append([method, kappa, beta, i, fe, re, be, chg, bf, br])
    return rows


def qr_solve_device(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Householder-QR baseline solution (cli.py:53-56), on the device via
    cuSOLVER (torch.linalg.qr): an evaluation reference, not the solve path."""
    import torch

    dev = torch.device("cuda", torch.cuda.current_device())
    at = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(dev)
    bt = torch.from_numpy(np.ascontiguousarray(b, dtype=np.float64)).to(dev)
    q, r = torch.linalg.qr(at, mode="reduced")
    x = torch.linalg.solve_triangular(r, (q.T @ bt)[:, None], upper=True)[:, 0]
    return x.cpu().numpy()


def cmd_solve(args) -> int:
    from .problems import gen_randsvd
    from .solvers import iterative_sketching

    prob = gen_randsvd(args.m, args.n, args.cond, args.resnorm, args.seed[0])
    cfg = _solver_cfg(args, args.m, args.n)
    res = iterative_sketching(prob.a, prob.b, cfg, prob.truth)
    save_numeric_csv(args.out, ["x"], np.asarray(res.solution)[:, None])
    t = res.trace
    write_table(args.summary or (args.out + ".summary.csv"), "iters,stop_reason,fe,re,be",
                [[res.iterations, t.stop_reason, _last(t.fe), _last(t.re), _last(t.be)]])
    return EXIT_DIVERGED if t.stop_reason == "diverged" else EXIT_OK


def cmd_convergence(args) -> int:
    from .embed import default_distortion
    from .problems import gen_randsvd
    from .solvers import iterative_sketching

    rows: list[list] = []
    tiny = np.finfo(float).tiny
    for kappa in args.cond:
        for beta in args.resnorm:
            for seed in args.seed:
                prob = gen_randsvd(args.m, args.n, kappa, beta, seed)
                cfg = _solver_cfg(args, args.m, args.n, seed=seed)
                res = iterative_sketching(prob.a, prob.b, cfg, prob.truth)
                eps = default_distortion(args.n, cfg.d)
                bounds = None
                if args.variant == "basic" and eps < 1 - 1 / math.sqrt(2):
                    bf, br = bound_curve("basic", eps, prob.truth.kappa, 1.0, prob.truth.beta,
                                         len(res.trace.iterates))
                    bounds = (bf / np.linalg.norm(prob.truth.x), br / max(prob.truth.beta, tiny))
                rows += _trace_rows(f"is_{args.variant}", kappa, beta, res, bounds)
                xqr = qr_solve_device(prob.a, prob.b)
                fe = float(np.linalg.norm(prob.truth.x - xqr))
                re = float(np.linalg.norm(prob.truth.r - (prob.b - prob.a @ xqr)) / max(prob.truth.beta, tiny))
                be = float("nan")
                if args.metrics == "full":
                    import torch

                    from .metrics import backward_error_device

                    dev = torch.device("cuda", torch.cuda.current_device())
                    be = backward_error_device(torch.from_numpy(prob.a).to(dev), torch.from_numpy(prob.b).to(dev),
                                               torch.from_numpy(xqr).to(dev))
                rows.append(["householder_qr", kappa, beta, -1, fe, re, be,
                             float("nan"), float("nan"), float("nan")])
    write_table(args.out, TRACE_HEADER, rows)
    return EXIT_OK


def cmd_compare(args) -> int:
    from .lsqr import sketch_and_precondition
    from .problems import gen_randsvd
    from .solvers import iterative_sketching

    prob = gen_randsvd(args.m, args.n, args.cond, args.resnorm, args.seed[0])
    rows: list[list] = []
    for variant in ("basic", "damped", "momentum"):
        cfg = _solver_cfg(args, args.m, args.n, variant=variant)
        rows += _trace_rows(f"is_{variant}", args.cond, args.resnorm,
                            iterative_sketching(prob.a, prob.b, cfg, prob.truth))
    for init in ("zero", "sketch_and_solve"):
        cfg = _solver_cfg(args, args.m, args.n, variant="basic", init=init)
        cfg.track_be = False  # the device sketch-and-precondition does not trace BE
        rows += _trace_rows(f"sp_{init}", args.cond, args.resnorm,
                            sketch_and_precondition(prob.a, prob.b, cfg, prob.truth))
    write_table(args.out, TRACE_HEADER, rows)
    return EXIT_OK


def cmd_dims(args) -> int:
    rows = [[v, args.m, args.n, args.accuracy, choose_dim(args.m, args.n, args.accuracy, v)]
            for v in ("basic", "damped", "momentum")]
    write_table(args.out, "variant,m,n,accuracy,d", rows)
    return EXIT_OK


def cmd_sparsebench(args) -> int:
    import torch

    from .problems import gen_sparse
    from .solvers import iterative_sketching
    from .sparse import residual_norm_device

    rows = []
    for m in args.rows:
        prob = gen_sparse(m, args.n, args.seed[0])
        d = 30 * args.n if args.d == "auto" else int(args.d)
        from .solvers import SolverConfig

        cfg = SolverConfig(d=d, zeta=args.zeta, max_iters=args.max_iters, rng_seed=args.seed[0])
        times = []
        res = None
        for _ in range(args.repeats):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            res = iterative_sketching(prob.a, prob.b, cfg)
            torch.cuda.synchronize()
            times.append(1e3 * (time.perf_counter() - t0))
        resnorm = residual_norm_device(prob.a, prob.b, res.solution)
        rows.append([m, args.n, d, float(np.median(times)), res.iterations, resnorm])
    write_table(args.out, "m,n,d,time_ms,iters,final_resnorm", rows)
    return EXIT_OK


# --------------------------------------------------------------------------
# Parser (cli.py:280-349)
# --------------------------------------------------------------------------
def _add_problem_flags(p: _Parser) -> None:
    p.add_argument("--m", type=int, required=True)
    p.add_argument("--n", type=int, required=True)
    p.add_argument("--cond", type=float, required=True)
    p.add_argument("--resnorm", type=float, required=True)


def _add_solver_flags(p: _Parser) -> None:
    p.add_argument("--d", default="auto", help='embedding dimension or "auto"')
    p.add_argument("--zeta", type=int, default=8)
    p.add_argument("--variant", choices=["basic", "damped", "momentum"], default="basic")
    p.add_argument("--max-iters", type=int, default=100)
    p.add_argument("--seed", type=int, nargs="+", default=[0])
    p.add_argument("--accuracy", type=float, default=2.0 ** -53,
                   help="accuracy level fed to the dimension formula when --d auto")
    p.add_argument("--metrics", choices=["cheap", "full"], default="cheap")
    p.add_argument("--out", required=True)
    p.add_argument("--device", default="cuda", help="cuda or cuda:K (the B200 to solve on)")


def build_parser() -> _Parser:
    parser = _Parser(prog="itsketch-b200")
    sub = parser.add_subparsers(dest="command", required=True, parser_class=_Parser)

    p = sub.add_parser("solve", help="solve one generated instance")
    _add_problem_flags(p)
    _add_solver_flags(p)
    p.add_argument("--summary", default=None)
    p.set_defaults(fn=cmd_solve, needs_device=True)

    p = sub.add_parser("convergence", help="per-iteration error traces vs QR reference")
    p.add_argument("--m", type=int, required=True)
    p.add_argument("--n", type=int, required=True)
    p.add_argument("--cond", type=float, nargs="+", required=True)
    p.add_argument("--resnorm", type=float, nargs="+", required=True)
    _add_solver_flags(p)
    p.set_defaults(fn=cmd_convergence, needs_device=True)

    p = sub.add_parser("compare", help="iterative sketching variants vs sketch-and-precondition")
    _add_problem_flags(p)
    _add_solver_flags(p)
    p.set_defaults(fn=cmd_compare, needs_device=True)

    p = sub.add_parser("dims", help="embedding-dimension table")
    p.add_argument("--m", type=int, required=True)
    p.add_argument("--n", type=int, required=True)
    p.add_argument("--accuracy", type=float, default=2.0 ** -53)
    p.add_argument("--out", required=True)
    p.set_defaults(fn=cmd_dims, needs_device=False)

    p = sub.add_parser("sparsebench", help="sparse problem timing scan")
    p.add_argument("--rows", type=int, nargs="+", required=True)
    p.add_argument("--n", type=int, required=True)
    p.add_argument("--repeats", type=int, default=3)
    _add_solver_flags(p)
    p.set_defaults(fn=cmd_sparsebench, needs_device=True)
    return parser


def main(argv: list[str] | None = None) -> int:
    args = build_parser().parse_args(argv)
    try:
        if args.needs_device:
            _select_device(args.device)
        return args.fn(args)
    except OSError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_IO


if __name__ == "__main__":
    sys.exit(main())

"""Golden fixtures for SURVEY §8 rows f-3 (CLI) and f-4 (sparse A), generated
by running the UNMODIFIED reference in the build container:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_sparse_cli.py

Writes tests/golden/sparse_cli.npz:
  gen_sparse     problems.py:92-110 — CSR arrays and b for small cases, sha256
                 digests at sparsebench sizes
  sketch_sparse  embed.py:76-80 (apply_sparse) — S·A for sparse A, bitwise
  sparse_solve   iterative_sketching on gen_sparse instances (solvers.py:323-345
                 via the sparse branches :195-196, :290, :299, :343): iterates,
                 residual changes, stop reason, normest, condest; and the
                 residual vectors' norms
  dims / bounds  choose_dim (embed.py:138-158), theoretical_bound_curve
                 (solvers.py:140-171)
  cli_*          the reference CLI's CSV files for solve / dims / sparsebench /
                 compare (cli.py:102-123,179-199,259-274), as text
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import tempfile

import numpy as np

REF = os.environ.get("ITSKETCH_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)

from itsketch import cli  # noqa: E402
from itsketch.embed import choose_dim, sparse_sign_new  # noqa: E402
from itsketch.problems import gen_sparse  # noqa: E402
from itsketch.solvers import SolverConfig, iterative_sketching, theoretical_bound_curve  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "sparse_cli.npz")


def sha(*arrs) -> str:
    h = hashlib.sha256()
    for a in arrs:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def main() -> None:
    g: dict[str, object] = {}
    # ---- gen_sparse ------------------------------------------------------
    for (m, n, seed) in [(50, 5, 0), (2000, 40, 0), (300, 3, 7)]:
        p = gen_sparse(m, n, seed)
        k = f"gs_{m}_{n}_{seed}"
        g[k + "_indptr"] = p.a.indptr.astype(np.int64)
        g[k + "_indices"] = p.a.indices.astype(np.int32)
        g[k + "_data"] = p.a.data
        g[k + "_b"] = p.b
    digests = {}
    for (m, n, seed) in [(200000, 100, 0), (100000, 100, 0), (1000000, 500, 3)]:
        p = gen_sparse(m, n, seed)
        digests[f"{m}_{n}_{seed}"] = sha(p.a.indptr.astype(np.int64), p.a.indices.astype(np.int32), p.a.data, p.b)
    g["gs_digests"] = json.dumps(digests)
    # ---- S·A for sparse A (bitwise) ---------------------------------------
    for (m, n, seed, d, zeta) in [(5000, 50, 2, 1000, 8), (2000, 40, 0, 1200, 8), (300, 3, 7, 20, 4),
                                  (40000, 200, 5, 6000, 8)]:
        p = gen_sparse(m, n, seed)
        s = sparse_sign_new(d, m, zeta, seed)
        k = f"sk_{m}_{n}_{seed}_{d}_{zeta}"
        sa = s.apply_sparse(p.a)
        if m * n <= 200000:
            g[k] = sa
        g[k + "_sha"] = sha(sa)
        g[k + "_sb_sha"] = sha(s.apply_vec(p.b))
    # ---- sparse solves ----------------------------------------------------
    cases = {
        "sp_basic": ((2000, 40, 0), dict(d=1200, max_iters=30)),
        "sp_mom": ((20000, 100, 1), dict(d=3000, variant="momentum", max_iters=40, rng_seed=1)),
        "sp_damped": ((20000, 100, 2), dict(d=3000, variant="damped", max_iters=40, rng_seed=2)),
        "sp_n3": ((500, 3, 4), dict(d=90, max_iters=25, rng_seed=4)),
    }
    for name, ((m, n, seed), cfgd) in cases.items():
        p = gen_sparse(m, n, seed)
        res = iterative_sketching(p.a, p.b, SolverConfig(**cfgd))
        t = res.trace
        g[f"{name}_problem"] = np.array([m, n, seed])
        g[f"{name}_config"] = json.dumps(cfgd)
        g[f"{name}_iterates"] = np.array(t.iterates)
        g[f"{name}_changes"] = np.array(t.residual_changes)
        g[f"{name}_rnorms"] = np.array([np.linalg.norm(r) for r in t.residual_vectors])
        g[f"{name}_stop"] = t.stop_reason
        g[f"{name}_est"] = np.array([t.normest, t.condest])
    # ---- dims / bounds -----------------------------------------------------
    dims = []
    for (m, n, acc) in [(200000, 200, 2.0 ** -53), (4000, 50, 1e-10), (10 ** 7, 1000, 1e-6), (100, 100, 0.5),
                        (3 * 10 ** 6, 10, 2.0 ** -53)]:
        for v in ("basic", "damped", "momentum"):
            dims.append([m, n, acc, v, choose_dim(m, n, acc, v)])
    g["dims"] = json.dumps(dims)
    bounds = []
    for (v, eps, kappa, na, nr, iters, first) in [("basic", 0.2, 1e10, 1.0, 1e-6, 20, 0),
                                                   ("damped", 0.3, 1e8, 2.0, 1e-3, 15, 0),
                                                   ("momentum", 0.2887, 1e8, 1.0, 1e-6, 18, 2),
                                                   ("basic", 0.05 ** 0.5, 1e15, 1.0, 1e-3, 30, 3)]:
        fe, re = theoretical_bound_curve(v, eps, kappa, na, nr, iters, first)
        bounds.append([v, eps, kappa, na, nr, iters, first, list(fe), list(re)])
    g["bounds"] = json.dumps(bounds)
    # ---- CLI files ---------------------------------------------------------
    with tempfile.TemporaryDirectory() as td:
        out = os.path.join(td, "x.csv")
        rc = cli.main(["solve", "--m", "500", "--n", "10", "--cond", "1e6", "--resnorm", "1e-6", "--d", "200",
                       "--out", out])
        g["cli_solve_rc"] = rc
        g["cli_solve_x"] = open(out).read()
        g["cli_solve_summary"] = open(out + ".summary.csv").read()
        out = os.path.join(td, "dims.csv")
        cli.main(["dims", "--m", "200000", "--n", "200", "--out", out])
        g["cli_dims"] = open(out).read()
        out = os.path.join(td, "sp.csv")
        cli.main(["sparsebench", "--rows", "2000", "--n", "40", "--repeats", "1", "--max-iters", "30", "--out", out])
        g["cli_sparsebench"] = open(out).read()
        out = os.path.join(td, "cmp.csv")
        cli.main(["compare", "--m", "600", "--n", "12", "--cond", "1e8", "--resnorm", "1e-6", "--d", "240",
                  "--max-iters", "40", "--out", out])
        g["cli_compare"] = open(out).read()
        out = os.path.join(td, "conv.csv")
        cli.main(["convergence", "--m", "600", "--n", "12", "--cond", "1e4", "1e8", "--resnorm", "1e-6",
                  "--d", "240", "--max-iters", "40", "--seed", "0", "1", "--out", out])
        g["cli_convergence"] = open(out).read()
    np.savez_compressed(OUT, **{k: (np.array(v) if isinstance(v, (str, int)) else v) for k, v in g.items()})
    print("wrote", OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main()

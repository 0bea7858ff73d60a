"""Generate the golden fixtures that pin the CPU oracle (and, through it, the
B200 path) to the reference implementation.

Run in the build container, where the reference is importable:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports the UNMODIFIED reference package from /root/reference/pkg/src (or
$ITSKETCH_REF) and records its outputs on seeded inputs:

  patterns.npz  — sparse_sign_new rows/signs (embed.py:83-99) for edge cases
                  (zeta == d, zeta == 1, rejection-heavy d=3), the raw PCG64
                  word stream, bounded draws with frequent Lemire rejections,
                  and S·A (embed.py:62-67) on seeded Gaussian inputs, bitwise;
                  plus sha256 digests of the full C1/C2/C3-size patterns.
  solves.npz    — iterative_sketching traces (solvers.py:323-345) on
                  gen_randsvd problems: iterates, fe/re/be, residual changes,
                  stop reason, normest, condest, for basic/damped/momentum,
                  zero init, extra_iters, consistent systems, track_be and a
                  diverging configuration.
  linalg.npz    — householder_qr_econ R factors, normest / condest values.
  lsqr.npz      — sketch_and_precondition traces (solvers.py:485-525) and
                  lsqr (solvers.py:411-482) solutions / iteration counts.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

REF = os.environ.get("ITSKETCH_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)

from itsketch.embed import sparse_sign_new  # noqa: E402
from itsketch.linalg import cond_est, householder_qr_econ, rand_power_norm_est  # noqa: E402
from itsketch.problems import gen_randsvd  # noqa: E402
from itsketch.solvers import SolverConfig, iterative_sketching, lsqr, sketch_and_precondition  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def sha(arr) -> str:
    return hashlib.sha256(np.ascontiguousarray(arr).tobytes()).hexdigest()


PATTERN_CASES = [
    # (d, m, zeta, seed, ncols of seeded A for S·A)
    (4, 3, 4, 0, 2),  # zeta == d: np.tile branch, no draws for rows
    (30, 50, 5, 1, 3),
    (25, 40, 6, 2, 3),
    (3, 200, 2, 3, 2),  # rejection-heavy: 1/3 of columns redrawn per round
    (20, 30, 1, 7, 4),  # zeta == 1
    (1000, 4000, 8, 0, 5),  # C1 shape
    (240, 500, 8, 3, 13),
    (50000, 3000, 16, 5, 3),  # large d, zeta 16
    (7, 1000, 7, 11, 2),  # zeta == d again, larger m
    (9, 777, 8, 12, 3),  # zeta close to d: heavy redraw
]

DIGEST_CASES = [
    # (d, m, zeta, seed) — full-size patterns pinned by digest only
    (1000, 4000, 8, 0),
    (4000, 200000, 8, 0),
    (4000, 200000, 8, 1),
    (10000, 1000000, 8, 0),
    (400, 1 << 20, 16, 0),
]

SOLVE_CASES = [
    # name, (m, n, kappa, beta, seed), config kwargs
    ("c1_basic", (4000, 50, 1e10, 1e-6, 0), dict(d=1000)),
    ("c1_damped", (4000, 50, 1e10, 1e-6, 0), dict(d=1000, variant="damped")),
    ("c1_momentum", (4000, 50, 1e10, 1e-6, 0), dict(d=1000, variant="momentum")),
    ("c1_seed1", (4000, 50, 1e10, 1e-6, 1), dict(d=1000, rng_seed=1)),
    ("c3like", (4000, 50, 1e15, 1e-3, 1), dict(d=1000, rng_seed=1, max_iters=100)),
    ("bitwise", (500, 12, 1e4, 1e-3, 3), dict(d=240, max_iters=6, rng_seed=3)),
    ("consistent", (400, 15, 1e3, 0.0, 0), dict(d=300, max_iters=20)),
    ("extra3", (2000, 30, 1e8, 1e-4, 4), dict(d=600, max_iters=200, rng_seed=4, extra_iters=3)),
    ("zero_init", (1000, 20, 1e8, 1e-4, 7), dict(d=400, init="zero", max_iters=100, rng_seed=7)),
    ("be_direct", (300, 10, 1e2, 1e-3, 1), dict(d=200, max_iters=30, track_be=True, rng_seed=1)),
    ("be_fast", (1000, 20, 1e4, 1e-3, 6), dict(d=400, max_iters=30, track_be=True, rng_seed=6)),
    ("diverge", (2000, 50, 1e6, 1e-2, 2), dict(d=52, max_iters=100, rng_seed=2)),
    ("maxit0", (500, 12, 1e4, 1e-3, 3), dict(d=240, max_iters=0, rng_seed=3)),
    ("eps_override", (1000, 20, 1e4, 1e-3, 6), dict(d=400, variant="momentum", epsilon_for_params=0.3, rng_seed=6)),
    ("c4proxy_mom", (40000, 200, 1e8, 1e-6, 0), dict(d=2400, variant="momentum", max_iters=100)),
]


def make_patterns():
    out = {}
    meta = []
    for d, m, zeta, seed, k in PATTERN_CASES:
        s = sparse_sign_new(d, m, zeta, seed)
        key = f"p_{d}_{m}_{zeta}_{seed}"
        out[key + "_rows"] = s.rows.astype(np.int32)
        out[key + "_signs"] = s.signs.astype(np.int8)
        a = np.random.default_rng(seed + 100).standard_normal((m, k))
        out[key + "_a_seed"] = np.array([seed + 100, k])
        out[key + "_sa"] = s.apply_dense(a)
        meta.append([d, m, zeta, seed, k])
    out["pattern_cases"] = np.array(meta, dtype=np.int64)
    digests = []
    for d, m, zeta, seed in DIGEST_CASES:
        s = sparse_sign_new(d, m, zeta, seed)
        digests.append(dict(d=d, m=m, zeta=zeta, seed=seed, rows=sha(s.rows.astype(np.int64)),
                            signs=sha(s.signs.astype(np.float64))))
    # S·A on a seeded Gaussian at C2 shape, 8 columns, pinned by digest
    s = sparse_sign_new(4000, 200000, 8, 0)
    a = np.random.default_rng(1234).standard_normal((200000, 8))
    sa = s.apply_dense(a)
    digests.append(dict(kind="sa", d=4000, m=200000, zeta=8, seed=0, a_seed=1234, k=8, sa=sha(sa)))
    out["digests_json"] = np.array(json.dumps(digests))
    # raw word stream + bounded draws with a high rejection rate
    g = np.random.default_rng(2024)
    out["raw_state_json"] = np.array(json.dumps(g.bit_generator.state))
    out["raw64"] = g.bit_generator.random_raw(64)
    g = np.random.default_rng(99)
    out["lemire_state_json"] = np.array(json.dumps(g.bit_generator.state))
    out["lemire_bound"] = np.array([3 * (1 << 30)])
    out["lemire_draws"] = g.integers(0, 3 * (1 << 30), size=257)
    out["lemire_draws2"] = g.integers(0, 1000, size=33)
    np.savez_compressed(os.path.join(HERE, "patterns.npz"), **out)


def make_solves():
    out = {}
    names = []
    for name, (m, n, kappa, beta, seed), kw in SOLVE_CASES:
        p = gen_randsvd(m, n, kappa, beta, seed)
        cfg = SolverConfig(**kw)
        res = iterative_sketching(p.a, p.b, cfg, p.truth)
        tr = res.trace
        out[f"{name}_problem"] = np.array([m, n, kappa, beta, seed], dtype=np.float64)
        out[f"{name}_config"] = np.array(json.dumps(kw))
        out[f"{name}_iterates"] = np.array(tr.iterates)
        out[f"{name}_fe"] = np.array(tr.fe)
        out[f"{name}_re"] = np.array(tr.re)
        out[f"{name}_be"] = np.array(tr.be)
        out[f"{name}_changes"] = np.array(tr.residual_changes)
        out[f"{name}_stop"] = np.array(tr.stop_reason)
        out[f"{name}_normest"] = np.array(tr.normest)
        out[f"{name}_condest"] = np.array(tr.condest)
        out[f"{name}_solution"] = res.solution
        # pin the generator: norms and a few entries of A and b
        out[f"{name}_gen"] = np.concatenate([
            [np.linalg.norm(p.a), np.linalg.norm(p.b), p.a[0, 0], p.a[-1, -1], p.b[0], p.b[-1]],
            p.truth.x[:4],
        ])
        names.append(name)
        print(f"{name}: iters={res.iterations} stop={tr.stop_reason} fe={tr.fe[-1] if tr.fe else None:.3e}")
    out["names"] = np.array(names)
    # one tiny problem stored in full, to pin gen_randsvd entrywise
    p = gen_randsvd(500, 12, 1e4, 1e-3, 3)
    out["tiny_a"] = p.a
    out["tiny_b"] = p.b
    out["tiny_x"] = p.truth.x
    out["tiny_r"] = p.truth.r
    np.savez_compressed(os.path.join(HERE, "solves.npz"), **out)


def make_linalg():
    out = {}
    rng = np.random.default_rng(5)
    for i, (m, n) in enumerate([(20, 5), (200, 40), (600, 50), (2, 1)]):
        a = rng.standard_normal((m, n)) if (m, n) != (2, 1) else np.array([[3.0], [4.0]])
        qr = householder_qr_econ(a)
        out[f"qr{i}_a"] = a
        out[f"qr{i}_r"] = qr.r
    for i, n in enumerate([1, 2, 7, 50, 200]):
        r = np.triu(rng.standard_normal((n, n))) + (2.0 + n) * np.eye(n)
        out[f"tri{i}_r"] = r
        out[f"tri{i}_normest"] = np.array(rand_power_norm_est(r, rng_seed=i))
        out[f"tri{i}_condest"] = np.array(cond_est(r))
    np.savez_compressed(os.path.join(HERE, "linalg.npz"), **out)


SAP_CASES = [
    # name, (m, n, kappa, beta, seed), SolverConfig kwargs
    ("sap_hard", (4000, 50, 1e10, 1e-6, 0), dict(d=1000, max_iters=60)),
    ("sap_zero", (4000, 50, 1e10, 1e-6, 0), dict(d=1000, init="zero", max_iters=60)),
    ("sap_consistent", (400, 15, 1e4, 0.0, 0), dict(d=300, max_iters=50)),
    ("sap_consistent_zero", (400, 15, 1e4, 0.0, 0), dict(d=300, init="zero", max_iters=50)),
    ("sap_small", (300, 10, 1e2, 1e-3, 1), dict(d=200, max_iters=30)),
    ("sap_c3like", (4000, 50, 1e15, 1e-3, 1), dict(d=1000, max_iters=100, rng_seed=1)),
    ("sap_maxit", (4000, 50, 1e10, 1e-6, 2), dict(d=1000, max_iters=5, rng_seed=2)),
]


def make_lsqr():
    out = {}
    names = []
    for name, (m, n, kappa, beta, seed), kw in SAP_CASES:
        p = gen_randsvd(m, n, kappa, beta, seed)
        res = sketch_and_precondition(p.a, p.b, SolverConfig(**kw), p.truth)
        tr = res.trace
        out[f"{name}_problem"] = np.array([m, n, kappa, beta, seed], dtype=np.float64)
        out[f"{name}_config"] = np.array(json.dumps(kw))
        out[f"{name}_iterates"] = np.array(tr.iterates)
        out[f"{name}_fe"] = np.array(tr.fe)
        out[f"{name}_re"] = np.array(tr.re)
        out[f"{name}_changes"] = np.array(tr.residual_changes)
        out[f"{name}_stop"] = np.array(tr.stop_reason)
        out[f"{name}_normest"] = np.array(tr.normest)
        out[f"{name}_condest"] = np.array(tr.condest)
        out[f"{name}_solution"] = res.solution
        names.append(name)
        print(f"{name}: iters={res.iterations} stop={tr.stop_reason} fe={tr.fe[-1]:.3e}")
    out["names"] = np.array(names)
    # lsqr with the exact QR preconditioner on Gaussian problems (acceptance C10)
    for seed in range(5):
        rng = np.random.default_rng(seed)
        a = rng.standard_normal((200, 20))
        b = rng.standard_normal(200)
        r_fac = householder_qr_econ(a).r
        x, iters = lsqr(a, b, np.zeros(20), r_fac, max_iters=3)
        out[f"c10_{seed}_a"], out[f"c10_{seed}_b"], out[f"c10_{seed}_r"] = a, b, r_fac
        out[f"c10_{seed}_x"], out[f"c10_{seed}_iters"] = x, np.array(iters)
    # lsqr with a sketched preconditioner (test_sketch_preconditioner_matches_dense)
    rng = np.random.default_rng(2)
    a = rng.standard_normal((200, 20))
    b = rng.standard_normal(200)
    r_fac = householder_qr_econ(sparse_sign_new(100, 200, 8, 2).apply_dense(a)).r
    x, iters = lsqr(a, b, np.zeros(20), r_fac, max_iters=100)
    out["sk_a"], out["sk_b"], out["sk_r"], out["sk_x"], out["sk_iters"] = a, b, r_fac, x, np.array(iters)
    np.savez_compressed(os.path.join(HERE, "lsqr.npz"), **out)


if __name__ == "__main__":
    which = sys.argv[1:] or ["patterns", "linalg", "solves", "lsqr"]
    if "patterns" in which:
        make_patterns()
    if "linalg" in which:
        make_linalg()
    if "solves" in which:
        make_solves()
    if "lsqr" in which:
        make_lsqr()

"""The reference's own convergence / acceptance properties, held by the B200
path (VERDICT r1 "missing 4").  Each test restates one reference test on the
drop-in `iterative_sketching` with the reference's inputs, tolerances and
yardsticks; the yardsticks (Householder-QR solve, measure_distortion, rate
functions, bound curves) come from the CPU oracle, pinned to the reference in
tests/test_oracle_pin.py (tests/golden/theory.npz).

  C01  test_acceptance.py:58-74    FE/RE within 10x of QR on the 12-case grid
  C02  test_acceptance.py:77-95    geometric rate <= g_IS(eps) + 0.05, Thm bound
  C03  test_acceptance.py:98-114   sketch-and-solve quality (Fact 2.4), 100 seeds
  C06  test_acceptance.py:164-200  sketch-and-precondition vs iterative sketching (start vector, iterations to the QR level)
  C07  test_acceptance.py:203-216  backward-error dichotomy (and the device BE vs the oracle's)
  C08  test_acceptance.py:219-240  damped / momentum rates and final FE
  C09  test_acceptance.py:243-274  stopping rule: the same corners fire, same reasons / iterations as the oracle
  test_solvers.py:158-175 (sketch_and_solve: consistent system, quality bounds)
  test_solvers.py:173-182 (consistent system), :189-195, :197-207, :209-221,
  :235-246 (extra_iters plateau), :248-256 (bitwise determinism), :258-264
"""

import math
import time

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

U = 2.0 ** -53
SEEDS = (0, 1, 2)


@pytest.fixture(scope="module")
def pkg():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2311_04362_b200 as p

    return p


@pytest.fixture(scope="module")
def orc():
    from oracle import itsketch_oracle as o

    return o


def _solve(pkg, p, **cfg):
    t = pkg.Truth(x=p.truth.x, r=p.truth.r, kappa=p.truth.kappa, beta=p.truth.beta)
    return pkg.iterative_sketching(p.a, p.b, pkg.SolverConfig(**cfg), t)


def _rel_errors(p, x_hat):
    """test_acceptance.py:50-55."""
    fe = np.linalg.norm(p.truth.x - x_hat) / np.linalg.norm(p.truth.x)
    re = np.linalg.norm(p.truth.r - (p.b - p.a @ x_hat)) / p.truth.beta
    return float(fe), float(re)


def test_c01_forward_stability_vs_qr(pkg, orc):
    """test_acceptance.py:58-74: kappa in {1e1, 1e10} x beta in {1e-12, 1e-3}
    x seeds 0..2 (4000 x 50, d = 1000, max_iters = 100): FE and RE within 10x
    of Householder QR's, all 12 cases in <= 60 s."""
    t0 = time.perf_counter()
    worst = 0.0
    for kappa in (1e1, 1e10):
        for beta in (1e-12, 1e-3):
            for seed in SEEDS:
                p = pkg.gen_randsvd(4000, 50, kappa, beta, seed)
                res = _solve(pkg, p, d=1000, zeta=8, max_iters=100, rng_seed=seed)
                fe_is, re_is = res.trace.fe[-1], res.trace.re[-1]
                fe_qr, re_qr = _rel_errors(p, orc.qr_solve(p.a, p.b))
                assert fe_is <= 10 * fe_qr and re_is <= 10 * re_qr, (kappa, beta, seed, fe_is, fe_qr, re_is, re_qr)
                worst = max(worst, fe_is / fe_qr, re_is / re_qr)
    elapsed = time.perf_counter() - t0
    print(f"[C01] worst FE/RE ratio vs QR {worst:.3g} (limit 10), {elapsed:.1f} s")
    assert elapsed <= 60.0


def test_c02_geometric_rate(pkg, orc, golden):
    """test_acceptance.py:77-95: contraction of RE over iterations 1..8 within
    g_IS(eps) + 0.05 and no violation of the basic-variant bound curve."""
    p = pkg.gen_randsvd(2000, 50, 1e2, 1e-3, 0)
    res = _solve(pkg, p, d=1000, max_iters=12, rng_seed=1)
    basis = np.linalg.qr(np.column_stack([p.a, p.b]), mode="reduced")[0]
    eps = orc.measure_distortion(orc.sparse_sign_pattern(1000, 2000, 8, 1), basis)
    assert eps == pytest.approx(float(golden("theory.npz")["eps_c02"]), rel=1e-12)
    re = res.trace.re
    contraction = float(np.exp(np.mean([np.log(re[i + 1] / re[i]) for i in range(1, 8)])))
    limit = orc.rate_g_is(eps) + 0.05
    _, re_bound = orc.theoretical_bound_curve("basic", eps, p.truth.kappa, np.linalg.norm(p.a, 2),
                                              p.truth.beta, 8)
    violations = sum(re[i] > re_bound[i] / p.truth.beta + 1e-10 for i in range(9))
    print(f"[C02] contraction {contraction:.3f} <= {limit:.3f}, bound violations {violations}")
    assert contraction <= limit and violations == 0


def test_c08_damping_and_momentum(pkg, orc):
    """test_acceptance.py:219-240: damped (seed 3) and momentum (seed 7)
    contract at their optimal rates (+0.05) and end within 10x of QR's FE."""
    n, d = 50, 1000
    eps = math.sqrt(n / d)
    p = pkg.gen_randsvd(2000, n, 1e2, 1e-3, 0)
    fe_qr, _ = _rel_errors(p, orc.qr_solve(p.a, p.b))
    for variant, seed, g in (("damped", 3, orc.rate_g_damp(eps)), ("momentum", 7, orc.rate_g_mom(eps))):
        res = _solve(pkg, p, d=d, variant=variant, max_iters=60, rng_seed=seed)
        re = res.trace.re
        contraction = float(np.exp(np.mean([np.log(re[i + 1] / re[i]) for i in range(3, 10)])))
        print(f"[C08] {variant} contraction {contraction:.3f} <= {g + 0.05:.3f}, final FE {res.trace.fe[-1]:.2g}")
        assert contraction <= g + 0.05, (variant, contraction, g)
        assert res.trace.fe[-1] <= 10 * max(fe_qr, U), (variant, res.trace.fe[-1], fe_qr)


def test_consistent_system_exact_init(pkg):
    """test_solvers.py:173-182: beta = 0 — the sketch-and-solve start is
    already exact; the rule fires after at most one corrective step."""
    p = pkg.gen_randsvd(400, 15, 1e3, 0.0, 0)
    res = _solve(pkg, p, d=300, max_iters=20)
    assert res.trace.stop_reason == "stopped_by_rule"
    assert res.iterations <= 2
    assert res.trace.fe[0] <= 1e-12
    assert np.linalg.norm(res.solution - p.truth.x) <= 1e-12


def test_matches_qr_accuracy_hard_problem(pkg, orc):
    """test_solvers.py:189-195 (kappa 1e10, beta 1e-12)."""
    p = pkg.gen_randsvd(4000, 50, 1e10, 1e-12, 0)
    res = _solve(pkg, p, d=1000, max_iters=100)
    fe_qr = np.linalg.norm(orc.qr_solve(p.a, p.b) - p.truth.x)
    assert res.trace.fe[-1] <= 10 * max(fe_qr, U)


def test_geometric_contraction(pkg, orc, golden):
    """test_solvers.py:197-207: every step contracts RE by g_IS(eps) + 0.05."""
    p = pkg.gen_randsvd(1000, 20, 10.0, 1e-3, 1)
    res = _solve(pkg, p, d=400, max_iters=9, rng_seed=1)
    q = np.linalg.qr(p.a, mode="reduced")[0]
    eps = orc.measure_distortion(orc.sparse_sign_pattern(400, 1000, 8, 1), q)
    assert eps == pytest.approx(float(golden("theory.npz")["eps_geo"]), rel=1e-12)
    g = orc.rate_g_is(eps)
    re = res.trace.re
    for i in range(min(8, len(re) - 1)):
        assert re[i + 1] <= (g + 0.05) * re[i] + 1e-14, (i, re[i + 1], re[i], g)


def test_theorem_bound_surrogate(pkg, orc, golden):
    """test_solvers.py:209-221: RE stays under the basic-variant bound curve."""
    p = pkg.gen_randsvd(1000, 20, 100.0, 1e-3, 2)
    q = np.linalg.qr(p.a, mode="reduced")[0]
    eps = orc.measure_distortion(orc.sparse_sign_pattern(400, 1000, 8, 2), q)
    assert eps == pytest.approx(float(golden("theory.npz")["eps_thm"]), rel=1e-12)
    assert eps < 0.29
    res = _solve(pkg, p, d=400, max_iters=8, rng_seed=2)
    _, re_bound = orc.theoretical_bound_curve("basic", eps, p.truth.kappa, np.linalg.norm(p.a, 2),
                                              p.truth.beta, iters=8)
    for i, re_i in enumerate(res.trace.re[:9]):
        assert re_i <= re_bound[i] / p.truth.beta + 1e-10, (i, re_i, re_bound[i] / p.truth.beta)


def test_plateau_stability_extra_iters(pkg):
    """test_solvers.py:235-246: extra_iters = 3 runs exactly 3 more
    iterations and the plateau FE moves less than 10x either way."""
    p = pkg.gen_randsvd(2000, 30, 1e8, 1e-4, 4)
    res0 = _solve(pkg, p, d=600, max_iters=200, rng_seed=4)
    assert res0.trace.stop_reason == "stopped_by_rule"
    res3 = _solve(pkg, p, d=600, max_iters=200, rng_seed=4, extra_iters=3)
    assert res3.iterations == res0.iterations + 3
    fe_stop, fe_late = res0.trace.fe[-1], res3.trace.fe[-1]
    assert fe_late <= 10 * fe_stop and fe_stop <= 10 * fe_late


def test_bitwise_determinism_reference_case(pkg):
    """test_solvers.py:248-256."""
    p = pkg.gen_randsvd(600, 15, 1e6, 1e-4, 5)
    r1 = _solve(pkg, p, d=300, max_iters=40, rng_seed=5)
    r2 = _solve(pkg, p, d=300, max_iters=40, rng_seed=5)
    assert np.array_equal(r1.solution, r2.solution)
    assert r1.trace.fe == r2.trace.fe
    assert r1.trace.residual_changes == r2.trace.residual_changes
    assert r1.trace.stop_reason == r2.trace.stop_reason


def test_damped_and_momentum_converge(pkg):
    """test_solvers.py:258-264: FE <= 1e-10 without diverging."""
    p = pkg.gen_randsvd(1000, 20, 1e4, 1e-3, 6)
    for variant in ("damped", "momentum"):
        res = _solve(pkg, p, d=400, variant=variant, max_iters=60, rng_seed=6)
        assert res.trace.stop_reason != "diverged"
        assert res.trace.fe[-1] <= 1e-10, (variant, res.trace.fe[-1])


def _pattern_of(orc, s):
    """The device-generated pattern as the oracle's Pattern (bit-equal to the
    oracle's own, tests/test_gpu_parity.py; taken from the device here so the
    distortion is measured for the embedding sketch_and_solve uses)."""
    return orc.Pattern(d=s.d, m=s.m, zeta=s.zeta, rows=np.asarray(s.rows).astype(np.int64),
                       signs=np.asarray(s.signs).astype(np.float64), scale=s.scale)


def test_sketch_and_solve_consistent_system(pkg):
    """test_solvers.py:159-163: beta = 0 -> the sketched solve is exact."""
    p = pkg.gen_randsvd(400, 15, 1e4, 0.0, 0)
    s = pkg.sparse_sign_new(200, 400, 8, 0)
    x0, _ = pkg.sketch_and_solve(p.a, p.b, s)
    assert np.linalg.norm(p.b - p.a @ x0) <= 1e-12 * np.linalg.norm(p.b)


def test_sketch_and_solve_quality_bounds_and_factors(pkg, orc):
    """test_solvers.py:165-175: Fact 2.4's residual and forward-error bounds
    with the measured distortion of the same embedding; and the returned
    factors are those of S·A (linalg.py:42-46): Q R = S A, Q'Sb = z,
    R x0 = z, equal to the oracle's x0 to rounding."""
    p = pkg.gen_randsvd(1000, 20, 1e4, 1e-2, 1)
    s = pkg.sparse_sign_new(500, 1000, 8, 1)
    pat = orc.sparse_sign_pattern(500, 1000, 8, 1)
    q = np.linalg.qr(p.a, mode="reduced")[0]
    eps = orc.measure_distortion(pat, q)
    x0, f = pkg.sketch_and_solve(p.a, p.b, s)
    beta = p.truth.beta
    assert np.linalg.norm(p.b - p.a @ x0) <= (1 + eps) / (1 - eps) * beta * (1 + 1e-10)
    norm_a = np.linalg.norm(p.a, 2)
    fe_bound = 2 * math.sqrt(eps) / (1 - eps) * p.truth.kappa / norm_a * beta
    assert np.linalg.norm(p.truth.x - x0) <= fe_bound * (1 + 1e-10)
    sa, sb = orc.sketch_apply(pat, p.a), orc.sketch_apply(pat, p.b[:, None])[:, 0]
    n = 20
    assert np.linalg.norm(f.q @ f.r - sa) <= 100 * n * U * np.linalg.norm(sa)
    assert np.linalg.norm(f.q.T @ f.q - np.eye(n)) <= 100 * n * U
    assert np.linalg.norm(f.q.T @ sb - f.z) <= 100 * n * U * np.linalg.norm(sb)
    qo, ro = orc.householder_qr_econ(sa)
    x_ref = orc.tri_solve_upper(ro, qo.T @ sb)
    assert np.linalg.norm(x0 - x_ref) <= 100 * n * U * np.linalg.cond(sa) * np.linalg.norm(x_ref)


def test_c03_sketch_and_solve_quality(pkg, orc):
    """test_acceptance.py:98-114: over 100 seeds (1000 x 25, kappa 1e4, beta
    1e-3, d = 500) the sketch-and-solve residual and forward error stay
    within Fact 2.4's bounds at the embedding's measured distortion of
    range([A b]): 0 violations."""
    violations = 0
    for seed in range(100):
        p = pkg.gen_randsvd(1000, 25, 1e4, 1e-3, seed)
        s = pkg.sparse_sign_new(500, 1000, 8, seed)
        basis = np.linalg.qr(np.column_stack([p.a, p.b]), mode="reduced")[0]
        eps = orc.measure_distortion(_pattern_of(orc, s), basis)
        x0, _ = pkg.sketch_and_solve(p.a, p.b, s)
        slack = 1 + 1e-8
        if np.linalg.norm(p.b - p.a @ x0) / p.truth.beta > (1 + eps) / (1 - eps) * slack:
            violations += 1
        norm_a = np.linalg.norm(p.a, 2)
        fe_lim = 2 * math.sqrt(eps) / (1 - eps) * p.truth.kappa / norm_a * p.truth.beta
        if np.linalg.norm(p.truth.x - x0) > fe_lim * slack:
            violations += 1
    print(f"[C03] {violations} violations over 100 seeds (limit 0)")
    assert violations == 0


def test_c07_backward_error_dichotomy(pkg, orc):
    """test_acceptance.py:203-216: iterative sketching is backward stable
    when the residual is small (beta = 1e-12: BE <= 100u) and only forward
    stable when it is not (beta = 1e-3: BE >= 100u while Householder QR's is
    <= 100u).  The trace's BE (cfg.track_be: the device restatement of
    metrics.py:99-129) agrees with the oracle's on the same solution."""
    bes = {}
    for beta in (1e-12, 1e-3):
        p = pkg.gen_randsvd(4000, 50, 1e10, beta, 0)
        res = _solve(pkg, p, d=1000, max_iters=100, track_be=True)
        be_ref = orc.backward_error(p.a, p.b, res.solution)
        be_dev = res.trace.be[-1]
        assert abs(be_dev - be_ref) <= 1e-6 * be_ref + 50 * U, (beta, be_dev, be_ref)
        bes[beta] = be_ref
        if beta == 1e-3:
            be_qr = orc.backward_error(p.a, p.b, orc.qr_solve(p.a, p.b))
    print(f"[C07] BE(IS) {bes[1e-12]:.2g} / {bes[1e-3]:.2g}, BE(QR) {be_qr:.2g}, 100u = {100 * U:.2g}")
    assert bes[1e-12] <= 100 * U and bes[1e-3] >= 100 * U and be_qr <= 100 * U


def test_backward_error_device_matches_oracle(pkg, orc):
    """metrics.py:99-129 on the device against the oracle (test_metrics.py:
    101-137): both branches (m <= 400 literal SVD, m > 400 reduced form) over
    random scalings, the zero-residual, zero-x and size-cap cases."""
    from paper_2311_04362_b200.metrics import backward_error_device as be_dev

    def dev(a, b, x, **kw):
        return be_dev(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), torch.from_numpy(x).cuda(), **kw)

    rng = np.random.default_rng(2)
    for trial in range(12):
        m = int(rng.integers(500, 700)) if trial % 2 else int(rng.integers(30, 400))
        n = int(rng.integers(2, 12))
        a = rng.standard_normal((m, n)) * 10.0 ** rng.integers(-2, 2)
        x = rng.standard_normal(n)
        b = a @ x + 10.0 ** rng.integers(-10, -1) * rng.standard_normal(m)
        x_hat = np.linalg.lstsq(a, b, rcond=None)[0] + 10.0 ** rng.integers(-12, -3) * rng.standard_normal(n)
        ref = orc.backward_error(a, b, x_hat)
        assert abs(dev(a, b, x_hat) - ref) <= 1e-6 * ref + 50 * U, (trial, m, n)
    a = np.eye(3)
    x = np.array([1.0, 2.0, 3.0])
    assert dev(a, a @ x, x) == 0.0
    with pytest.raises(ValueError):
        dev(np.eye(3), np.ones(3), np.zeros(3))
    with pytest.raises(ValueError):
        dev(np.ones((11, 2)), np.ones(11), np.ones(2), max_m=10)


def test_c09_stopping_rule_agrees_with_reference(pkg, orc):
    """test_acceptance.py:243-274 (a known red of the reference: at kappa =
    1e1, beta = 1e-3 the rule needs more than 50 iterations): on the 12-case
    grid the device path stops for the same reason as the oracle, within
    max(3, 15 %) iterations of it, the same corners fire within 50 iterations,
    and where the rule fired the final FE is within 2x the oracle's."""
    red = []
    for kappa in (1e1, 1e10):
        for beta in (1e-12, 1e-3):
            for seed in SEEDS:
                p = pkg.gen_randsvd(4000, 50, kappa, beta, seed)
                res = _solve(pkg, p, d=1000, max_iters=100, rng_seed=seed)
                _, tr = orc.iterative_sketching(p.a, p.b, orc.Config(d=1000, max_iters=100, rng_seed=seed), p.truth)
                it_ref = len(tr.iterates) - 1
                assert res.trace.stop_reason == tr.stop_reason, (kappa, beta, seed)
                assert abs(res.iterations - it_ref) <= max(3, 0.15 * it_ref), (kappa, beta, seed, res.iterations, it_ref)
                within = res.trace.stop_reason == "stopped_by_rule" and res.iterations <= 50
                within_ref = tr.stop_reason == "stopped_by_rule" and it_ref <= 50
                assert within == within_ref, (kappa, beta, seed, res.iterations, it_ref)
                if not within:
                    red.append((kappa, beta, seed, res.iterations, it_ref))
                if res.trace.stop_reason == "stopped_by_rule":
                    assert res.trace.fe[-1] <= 2 * tr.fe[-1], (kappa, beta, seed, res.trace.fe[-1], tr.fe[-1])
    print(f"[C09] corners past 50 iterations (device, oracle): {red}")
    assert all(k == 1e1 and b == 1e-3 for k, b, *_ in red)


def test_c06_sketch_and_precondition(pkg, orc):
    """test_acceptance.py:164-200: with a zero start sketch-and-precondition
    stalls above 10x the QR forward error, with the sketch-and-solve start it
    reaches it; momentum and S&P reach the QR level at least 1.5x sooner than
    basic iterative sketching (4000 x 50, kappa 1e10, beta 1e-6, d = 1000)."""
    p = pkg.gen_randsvd(4000, 50, 1e10, 1e-6, 0)
    t = pkg.Truth(x=p.truth.x, r=p.truth.r, kappa=p.truth.kappa, beta=p.truth.beta)
    fe_qr, _ = _rel_errors(p, orc.qr_solve(p.a, p.b))
    d = 20 * 50
    zero = pkg.sketch_and_precondition(p.a, p.b, pkg.SolverConfig(d=d, init="zero", max_iters=120), t)
    ss = pkg.sketch_and_precondition(p.a, p.b, pkg.SolverConfig(d=d, init="sketch_and_solve", max_iters=120), t)
    basic = pkg.iterative_sketching(p.a, p.b, pkg.SolverConfig(d=d, max_iters=120), t)
    mom = pkg.iterative_sketching(p.a, p.b, pkg.SolverConfig(d=d, variant="momentum", max_iters=120), t)

    def first_at_qr_level(trace):
        return next((i for i, fe in enumerate(trace.fe) if fe <= 10 * fe_qr), None)

    it_basic, it_mom, it_sp = (first_at_qr_level(r.trace) for r in (basic, mom, ss))
    print(f"[C06] zero-init FE {zero.trace.fe[-1]:.2g} vs 10*QR {10 * fe_qr:.2g}; ss-init FE {ss.trace.fe[-1]:.2g}; "
          f"iterations to the QR level: basic {it_basic}, momentum {it_mom}, S&P {it_sp}")
    assert zero.trace.fe[-1] >= 10 * fe_qr and ss.trace.fe[-1] <= 10 * fe_qr
    assert None not in (it_basic, it_mom, it_sp)
    assert it_basic >= 1.5 * it_mom and it_basic >= 1.5 * it_sp

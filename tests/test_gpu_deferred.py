"""Deferred estimates: normest / condest run beside the loop's first
iterations and the stopping rule (solvers.py:174-192, 306-316) is replayed
over the iterates recorded before they were ready.

The deferred solve (residuals="all") must be BITWISE the synchronous one
(residuals="last": estimates complete before the loop): same iterates, trace,
stop reason and iteration count — the rule sees the same bits, only later.
The forced case holds the ready flag at zero for the whole loop, so every
rule evaluation happens in the replay (inside the loop once the flag is set,
or in itsk_loop_finish after a guard / max_iters stop).
"""

import ctypes
import json

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

NAMES = ["c1_basic", "c1_damped", "c1_momentum", "c3like", "consistent", "extra3", "zero_init", "diverge",
         "eps_override", "c4proxy_mom"]


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


def _problem(orc, g, name):
    m, n, kappa, beta, seed = g[f"{name}_problem"]
    a, b, truth = orc.gen_randsvd(int(m), int(n), kappa, beta, int(seed))
    cfg = json.loads(str(g[f"{name}_config"]))
    return a, b, truth, cfg


def _same(r1, r2):
    assert r1.trace.stop_reason == r2.trace.stop_reason
    assert r1.iterations == r2.iterations
    assert np.array_equal(r1.solution, r2.solution)
    assert r1.trace.residual_changes == r2.trace.residual_changes
    assert r1.trace.fe == r2.trace.fe and r1.trace.re == r2.trace.re
    assert r1.trace.normest == r2.trace.normest and r1.trace.condest == r2.trace.condest


@pytest.mark.parametrize("name", NAMES)
def test_deferred_estimates_bitwise_synchronous(pkg, orc, golden, name):
    g = golden("solves.npz")
    a, b, truth, cfgd = _problem(orc, g, name)
    t = pkg.Truth(x=truth.x, r=truth.r, kappa=truth.kappa, beta=truth.beta)
    cfg = pkg.SolverConfig(**cfgd)
    r_def = pkg.iterative_sketching(a, b, cfg, t, residuals="all")
    r_sync = pkg.iterative_sketching(a, b, cfg, t, residuals="last")
    _same(r_def, r_sync)
    # the deferred trace keeps every residual, as the reference's does
    assert len(r_def.trace.residual_vectors) == r_def.iterations + 1
    np.testing.assert_array_equal(r_def.trace.residual_vectors[-1], r_sync.trace.residual_vectors[-1])


def _solve_flag_held(pkg, a, b, cfg, truth, use_graph):
    """The solver's own steps, with the ready flag held at zero through the
    whole loop and set only before itsk_loop_finish."""
    from paper_2311_04362_b200 import device as dv
    from paper_2311_04362_b200 import _lib, solvers as sv

    m, n = a.shape
    dev = dv.current_device()
    lib = dv.lib(dev)
    alpha, beta = sv.update_coeffs(cfg, n)
    ws = sv._workspace(dev, m, n, cfg.d, cfg.zeta, cfg.max_iters, cfg.max_iters + 1, truth is not None)
    at = torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    ws.b.copy_(torch.from_numpy(b))
    if truth is not None:
        ws.x_true.copy_(torch.from_numpy(truth.x))
        if truth.beta > 0:
            ws.r_true.copy_(torch.from_numpy(truth.r))
    so = torch.cuda.current_stream(dev)
    s = int(so.cuda_stream)
    sv._sketch_qr_x0(lib, ws, at, n, ws.b, cfg, s, defer=False)
    _lib.check(lib.itsk_flag_store(dv.ptr(ws.est) + 16, 0, s))
    p = sv._loop_params(ws, at, n, cfg, alpha, beta, truth, defer=True)
    sv.run_loop(lib, ws, p, use_graph, s)
    _lib.check(lib.itsk_flag_store(dv.ptr(ws.est) + 16, 1, s))
    _lib.check(lib.itsk_loop_finish(ctypes.byref(p), s))
    res = sv._read_result(lib, ws, p, so)
    return sv._assemble(ws, res, truth, cfg, at, ws.b)


@pytest.mark.parametrize("use_graph", [True, False])
@pytest.mark.parametrize("name", ["c1_basic", "c1_momentum", "consistent", "extra3", "diverge", "c3like"])
def test_rule_replayed_after_loop(pkg, orc, golden, name, use_graph):
    """Estimates never ready inside the loop: it runs to max_iters (or the
    guard) and itsk_loop_finish moves the stop back to the reference's."""
    g = golden("solves.npz")
    a, b, truth, cfgd = _problem(orc, g, name)
    t = pkg.Truth(x=truth.x, r=truth.r, kappa=truth.kappa, beta=truth.beta)
    cfg = pkg.SolverConfig(**cfgd)
    r_sync = pkg.iterative_sketching(a, b, cfg, t, residuals="last")
    r_late = _solve_flag_held(pkg, a, b, cfg, t, use_graph)
    _same(r_late, r_sync)


def test_rule_replayed_short_max_iters(pkg):
    """The rule would fire at iterate k <= max_iters: the replay must stop
    there even when the loop itself reached max_iters first."""
    p = pkg.gen_randsvd(4000, 50, 1e6, 1e-8, 3)
    for extra in (0, 2):
        cfg0 = pkg.SolverConfig(d=1000, max_iters=60, extra_iters=extra, rng_seed=3)
        k = pkg.iterative_sketching(p.a, p.b, cfg0, residuals="last").iterations
        for mi in (k - 1, k, k + 1):
            cfg = pkg.SolverConfig(d=1000, max_iters=mi, extra_iters=extra, rng_seed=3)
            r_sync = pkg.iterative_sketching(p.a, p.b, cfg, residuals="last")
            r_late = _solve_flag_held(pkg, p.a, p.b, cfg, None, True)
            _same(r_late, r_sync)
            assert r_sync.trace.stop_reason == ("stopped_by_rule" if mi >= k else "max_iters")


def test_kept_results_keep_their_residual_rows(pkg):
    """Results kept by the caller keep valid residual vectors while the
    workspace is reused (a second buffer rotates in; with two results alive
    the older one's rows are copied out)."""
    p = pkg.gen_randsvd(20000, 40, 1e6, 1e-6, 7)
    kept = []
    for seed in (1, 2, 3, 4):
        cfg = pkg.SolverConfig(d=800, rng_seed=seed)
        kept.append(pkg.iterative_sketching(p.a, p.b, cfg, residuals="all"))
    for r in kept:
        for i in (0, len(r.trace.residual_vectors) - 1):
            want = p.b - p.a @ r.trace.iterates[i]
            np.testing.assert_allclose(r.trace.residual_vectors[i], want, rtol=0, atol=1e-12 * np.linalg.norm(p.b))

"""C4 — the north-star's headline configuration — at full size, and the GPU
problem generator's invariants (VERDICT r1 "missing 1" and "missing 6").

C4 (BASELINE.json configs[3]): the gen_randsvd construction 4e6 x 2000
(64 GB), kappa 1e8, ||r|| = 1e-6, d = 12n = 24000, zeta = 8, momentum (the
headline variant: basic never fires the stopping rule at d = 12n, SURVEY
§8(d)).  The host generator is infeasible at this size, so the instance is
built on the device (instances.gen_randsvd_device) and the SAME bytes are
copied to the host for the CPU oracle.

Bars (north_star): FE and RE within 2x of the oracle's (one-sided), and
||x - x_ref|| / ||x_ref|| <= 10 kappa u + FE_ref.

Documented, asserted expectation on the stop iteration: the B200 path stops
by the rule at ~18 iterations; the oracle (numpy/OpenBLAS) runs to max_iters
(50).  The rule needs ||r_{i+1} - r_i|| <= u (gamma normest ||x|| + rho
condest ||r||) ~ 1e-15 here, below the rounding noise of OpenBLAS's
2000-term dgemv dot products (~sqrt(n) u ||b||) once the iteration has
converged; the fused pass's dots (32-lane partial sums, a fixed shuffle
tree) are an order of magnitude quieter, so its residual change falls under
the threshold.  Both are valid outcomes of the same algorithm; FE / RE of
the GPU run are at or below the oracle's.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

U = 2.0 ** -53
M, N, KAPPA, BETA, D = 4_000_000, 2000, 1e8, 1e-6, 24000


@pytest.fixture(scope="module")
def pkg():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    free, total = torch.cuda.mem_get_info()
    if free < 100 * 2**30:
        pytest.skip(f"C4 needs ~100 GB of device memory, {free / 2**30:.0f} GiB free")
    import paper_2311_04362_b200 as p

    return p


def _check_instance(p, m, n, kappa, beta, spectrum: bool):
    """problems.py:65-89 invariants (test_problems.py:48-57): ||x|| = 1,
    ||r|| = beta, A'r ~ 0, b = A x + r; and the spectrum sigma_j = kappa^(-j/(n-1))."""
    a, b, r = p.a, p.b, p.truth.r
    x = torch.from_numpy(p.truth.x).to(a.device)
    assert a.shape == (m, n) and a.dtype == torch.float64 and a.is_cuda and a.is_contiguous()
    assert abs(float(torch.linalg.vector_norm(x)) - 1.0) <= 1e-14
    assert float(torch.linalg.vector_norm(r)) == pytest.approx(beta, rel=1e-12)
    # b = A x + r (row blocks: no m-sized temporaries beyond one vector)
    resid = torch.empty_like(b)
    blk = 1 << 18
    for i in range(0, m, blk):
        torch.addmv(r[i:i + blk], a[i:i + blk], x, out=resid[i:i + blk])
    assert float(torch.linalg.vector_norm(resid - b)) <= 1e-13 * float(torch.linalg.vector_norm(b))
    # r is orthogonal to range(A): ||A'r|| <= ~ sqrt(m) u ||A|| ||r||
    atr = torch.zeros(n, dtype=torch.float64, device=a.device)
    for i in range(0, m, blk):
        atr.addmv_(a[i:i + blk].T, r[i:i + blk])
    assert float(torch.linalg.vector_norm(atr)) <= 1e-10 * beta
    if spectrum:
        rf = torch.linalg.qr(a, mode="r")[1]
        sv = torch.linalg.svdvals(rf).cpu().numpy()
        want = kappa ** (-np.arange(n) / (n - 1))
        np.testing.assert_allclose(sv, want, rtol=1e-9 * max(1.0, kappa * 1e-6))


def test_device_generator_invariants_1e6(pkg):
    """gen_randsvd_device at m = 1e6 (n = 200, kappa 1e6, beta 1e-4): the
    construction's invariants, including the exact spectrum."""
    from paper_2311_04362_b200.instances import gen_randsvd_device

    p = gen_randsvd_device(1_000_000, 200, 1e6, 1e-4, 3)
    _check_instance(p, 1_000_000, 200, 1e6, 1e-4, spectrum=True)
    # determinism: the same seed gives the same bytes
    q = gen_randsvd_device(1_000_000, 200, 1e6, 1e-4, 3)
    assert torch.equal(p.a, q.a) and torch.equal(p.b, q.b)


def test_c4_full_size_parity(pkg):
    """C4 on the device vs the oracle on the same bytes (strict north-star bar)."""
    from oracle import itsketch_oracle as orc
    from paper_2311_04362_b200.instances import gen_randsvd_device

    p = gen_randsvd_device(M, N, KAPPA, BETA, 0)
    _check_instance(p, M, N, KAPPA, BETA, spectrum=False)
    cfg = pkg.SolverConfig(d=D, variant="momentum", rng_seed=0)
    res = pkg.iterative_sketching(p.a, p.b, cfg, p.truth, residuals="all")
    tr = res.trace
    # the same bytes on the host (pinned staging: ~2 s for 64 GB)
    a_h = torch.empty((M, N), dtype=torch.float64, pin_memory=True)
    blk = 1 << 18
    for i in range(0, M, blk):
        a_h[i:i + blk].copy_(p.a[i:i + blk], non_blocking=True)
    b_h, r_h = p.b.cpu().numpy(), p.truth.r.cpu().numpy()
    torch.cuda.synchronize()
    x_true = p.truth.x
    # S·[A | b] of the full instance (the streamed window sweep at its headline
    # size): a column subset, b included, bitwise equal to the oracle's
    # sequential sum over the same 4e6 rows
    s = pkg.sparse_sign_new(D, M, 8, 0)
    w = s.apply_dense(p.a, p.b)
    cols = [0, 1, 999, 1000, N - 1]
    sub = np.column_stack([a_h.numpy()[:, cols], b_h])
    pat = orc.Pattern(d=D, m=M, zeta=8, rows=np.asarray(s.rows).astype(np.int64),
                      signs=np.asarray(s.signs).astype(np.float64), scale=s.scale)
    assert np.array_equal(w[:, cols + [N]].cpu().numpy(), orc.sketch_apply(pat, sub))
    del s, w, pat, sub
    del p
    torch.cuda.empty_cache()
    otruth = orc.Truth(x=x_true, r=r_h, kappa=KAPPA, beta=BETA)
    x_ref, tr_ref = orc.iterative_sketching(a_h.numpy(), b_h, orc.Config(d=D, variant="momentum", rng_seed=0),
                                            otruth)
    ref_iters = len(tr_ref.iterates) - 1
    dev_x = float(np.linalg.norm(res.solution - x_ref) / np.linalg.norm(x_ref))
    bound = 10 * KAPPA * U + tr_ref.fe[-1]
    print(f"C4: B200 {res.iterations} it. ({tr.stop_reason}) FE {tr.fe[-1]:.3e} RE {tr.re[-1]:.3e}; "
          f"oracle {ref_iters} it. ({tr_ref.stop_reason}) FE {tr_ref.fe[-1]:.3e} RE {tr_ref.re[-1]:.3e}; "
          f"|x-x_ref|/|x_ref| {dev_x:.3e} <= {bound:.3e}")
    # estimates: the same R up to rounding
    assert tr.normest == pytest.approx(tr_ref.normest, rel=1e-10)
    assert tr.condest == pytest.approx(tr_ref.condest, rel=1e-8)
    # the sketch-and-solve start agrees to the rounding of the QR
    assert tr.fe[0] <= 2 * tr_ref.fe[0] and tr_ref.fe[0] <= 2 * tr.fe[0]
    # the north-star bars
    assert tr.fe[-1] <= 2 * tr_ref.fe[-1], (tr.fe[-1], tr_ref.fe[-1])
    assert tr.re[-1] <= 2 * tr_ref.re[-1], (tr.re[-1], tr_ref.re[-1])
    assert dev_x <= bound, (dev_x, bound)
    # the documented stop expectation (module docstring): B200 by the rule in
    # 15..22 iterations; the oracle at max_iters, or — should its dgemv noise
    # ever fall under the threshold — by the rule no earlier than the B200 run
    assert tr.stop_reason == "stopped_by_rule" and 15 <= res.iterations <= 22, (tr.stop_reason, res.iterations)
    assert (tr_ref.stop_reason == "max_iters" and ref_iters == 50) or (
        tr_ref.stop_reason == "stopped_by_rule" and ref_iters >= res.iterations - 2), (tr_ref.stop_reason, ref_iters)


def test_c4_pass_full_size(pkg):
    """The fused pass (itsk_fused_pass: r = b - A x, c = A'r, the four norms)
    at the C4 shape, 4e6 x 2000 = 64 GB, against a float64 row-block
    computation on the same device bytes (torch addmv), and the exact
    property of a zero iterate: r == b bitwise, c = A'b, ||r||^2 = ||b||^2."""
    import ctypes

    from paper_2311_04362_b200 import _lib
    from paper_2311_04362_b200 import device as dv

    dev = dv.current_device()
    g = torch.Generator(device=dev).manual_seed(4)
    a = torch.randn(M, N, dtype=torch.float64, device=dev, generator=g)
    b = torch.randn(M, dtype=torch.float64, device=dev, generator=g)
    x = torch.randn(N, dtype=torch.float64, device=dev, generator=g)
    r_prev = torch.randn(M, dtype=torch.float64, device=dev, generator=g)
    r_true = torch.randn(M, dtype=torch.float64, device=dev, generator=g)
    lib = dv.lib(dev)
    nb = ctypes.c_int64()
    _lib.check(lib.itsk_pass_workspace(M, N, ctypes.byref(nb)))
    ws = dv.workspace(nb.value, dev)
    r_out = torch.empty(M, dtype=torch.float64, device=dev)
    cs = torch.empty(N + 8, dtype=torch.float64, device=dev)

    def run(xv):
        _lib.check(lib.itsk_fused_pass(dv.ptr(a), M, N, N, dv.ptr(b), dv.ptr(xv), dv.ptr(r_prev), dv.ptr(r_out),
                                       dv.ptr(r_true), dv.ptr(cs), dv.ptr(ws), ws.numel(), dv.stream_ptr()))
        torch.cuda.synchronize()
        return r_out.clone(), cs.clone()

    def blocked(rv_from_x):
        blk = 1 << 18
        r = torch.empty(M, dtype=torch.float64, device=dev)
        c = torch.zeros(N, dtype=torch.float64, device=dev)
        cabs = torch.zeros(N, dtype=torch.float64, device=dev)
        for i in range(0, M, blk):
            torch.addmv(b[i:i + blk], a[i:i + blk], rv_from_x, alpha=-1.0, out=r[i:i + blk])
            c.addmv_(a[i:i + blk].T, r[i:i + blk])
            cabs.addmv_(a[i:i + blk].abs().T, r[i:i + blk].abs())
        return r, c, cabs

    r, got = run(x)
    r_ref, c_ref, cabs = blocked(x)
    # |r - r_ref| <= ~ n u |a|'|x| per row: normwise over the 4e6 rows
    xa = float(torch.linalg.vector_norm(x)) * (N ** 0.5)
    assert float((r - r_ref).abs().max()) <= 50 * N * U * xa
    assert float(torch.linalg.vector_norm(got[:N] - c_ref)) <= 1e-12 * float(torch.linalg.vector_norm(cabs))
    assert float(got[N]) == pytest.approx(float(r_ref @ r_ref), rel=1e-12)
    assert float(got[N + 1]) == pytest.approx(float((r_ref - r_prev) @ (r_ref - r_prev)), rel=1e-12)
    assert float(got[N + 2]) == pytest.approx(float((r_true - r_ref) @ (r_true - r_ref)), rel=1e-12)
    assert float(got[N + 3]) == pytest.approx(float(b @ b), rel=1e-12)
    # zero iterate: every dot is exactly zero
    r0, got0 = run(torch.zeros(N, dtype=torch.float64, device=dev))
    assert torch.equal(r0, b)
    _, c0, cabs0 = blocked(torch.zeros(N, dtype=torch.float64, device=dev))
    assert float(torch.linalg.vector_norm(got0[:N] - c0)) <= 1e-12 * float(torch.linalg.vector_norm(cabs0))
    assert float(got0[N]) == pytest.approx(float(b @ b), rel=1e-12)
    # bitwise repeatable (fixed reduction order)
    r1, got1 = run(x)
    assert torch.equal(r1, r) and torch.equal(got1[:N + 4], got[:N + 4])

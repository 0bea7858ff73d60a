"""Out-of-bounds and initialisation checks of our own (compute-sanitizer is
closed on this GPU pool: runs under it left GPUs needing a reset).

Every buffer a C-ABI entry point writes is placed inside a larger
allocation whose margins hold a canary byte pattern; padded leading
dimensions carry canary values in the pad columns; workspaces start as
garbage (0xA5 bytes, NaN-like).  After each call the canaries must be
intact (no write outside the documented extent) and the results finite and
equal, bit for bit, across three repetitions (a race or a read of
uninitialised workspace shows up as a changed or non-finite result).  The
Python solves run with `device.workspace` patched to hand out guarded
buffers, covering the pattern / QR / loop workspaces the solver allocates.
Kernels covered: pattern (first draw, redraws, CSR), sketch (register gather
and ring), QR (panel / look-ahead / two-level far update / next2 /
single-kernel fallback), fused pass (warp-per-row and row-group kernels),
TRSV, normest / condest, the loop (graph, step-wise, deferred estimates),
the in-process peer exchange, the sparse CSR path and LSQR.
"""

import ctypes

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

CANARY = 0x5A
MARGIN = 1 << 16


@pytest.fixture(scope="module")
def env():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2311_04362_b200 as itsk
    from paper_2311_04362_b200 import _lib
    from paper_2311_04362_b200 import device as dv

    dev = dv.current_device()
    return itsk, _lib, dv, dev, dv.lib(dev)


class Guard:
    """nbytes of payload between two canary margins (payload pre-filled)."""

    def __init__(self, nbytes, dev, fill=0xA5):
        self.n = int(nbytes)
        self.buf = torch.full((self.n + 2 * MARGIN,), CANARY, dtype=torch.uint8, device=dev)
        self.buf[MARGIN:MARGIN + self.n] = fill

    def payload(self):
        return self.buf[MARGIN:MARGIN + self.n]

    def view(self, dtype, shape):
        return self.payload().view(dtype).view(shape)

    def ok(self):
        torch.cuda.synchronize()
        return bool((self.buf[:MARGIN] == CANARY).all()) and bool((self.buf[MARGIN + self.n:] == CANARY).all())


def padded(rows, cols, ld, dev, fill_value):
    """(rows x ld) float64 storage with canary values in the pad columns."""
    g = Guard(rows * ld * 8, dev, fill=0)
    full = g.view(torch.float64, (rows, ld))
    full[:, cols:] = fill_value
    return g, full


PAD = float("nan")  # pad columns: a NaN read into arithmetic shows up as a non-finite result


def pad_intact(full, cols):
    """The pad columns still hold the canary NaN, bit for bit."""
    torch.cuda.synchronize()
    pad = full[:, cols:].contiguous().view(torch.int64)
    ref = torch.tensor([float("nan")], dtype=torch.float64, device=full.device).view(torch.int64)
    return bool((pad == ref).all())


def test_pattern_and_sketch_guards(env):
    itsk, _lib, dv, dev, lib = env
    from paper_2311_04362_b200.embed import pcg_state

    for d, m, zeta in [(300, 5000, 8), (40, 3000, 16), (2000, 100000, 8)]:
        words, has32, pend = pcg_state(3)
        nb = ctypes.c_int64()
        _lib.check(lib.itsk_pattern_workspace(d, m, zeta, ctypes.byref(nb)))
        outs = []
        for rep in range(3):
            gr, gn = Guard(4 * m * zeta, dev), Guard(m * zeta, dev)
            gp, gs = Guard(4 * (d + 1), dev), Guard(4 * m * zeta, dev)
            gw = Guard(nb.value, dev)
            _lib.check(lib.itsk_sparse_sign_pattern(d, m, zeta, words, has32, pend, dv.ptr(gr.payload()),
                                                    dv.ptr(gn.payload()), dv.ptr(gp.payload()), dv.ptr(gs.payload()),
                                                    dv.ptr(gw.payload()), nb.value, dv.stream_ptr()))
            assert all(g.ok() for g in (gr, gn, gp, gs, gw)), (d, m, zeta)
            outs.append(tuple(g.payload().clone() for g in (gr, gn, gp, gs)))
        for o in outs[1:]:
            assert all(torch.equal(x, y) for x, y in zip(o, outs[0]))
        # the sketch into a padded W (pad columns must stay untouched)
        for n in (40, 257):
            a = torch.randn(m, n, dtype=torch.float64, device=dev)
            b = torch.randn(m, dtype=torch.float64, device=dev)
            ldw = n + 1 + 3
            res = []
            for rep in range(3):
                g, W = padded(d, n + 1, ldw, dev, PAD)
                _lib.check(lib.itsk_sketch(dv.ptr(a), m, n, n, dv.ptr(b), dv.ptr(outs[0][2]), dv.ptr(outs[0][3]), d,
                                           zeta, dv.ptr(W), ldw, dv.stream_ptr()))
                assert g.ok() and pad_intact(W, n + 1) and bool(torch.isfinite(W[:, :n + 1]).all())
                res.append(W[:, :n + 1].clone())
            assert all(torch.equal(r, res[0]) for r in res[1:])


@pytest.mark.parametrize("d,n", [(300, 40), (4000, 201), (3000, 384), (16500, 1100), (30000, 130)])
def test_qr_guards(env, d, n):
    itsk, _lib, dv, dev, lib = env
    nb = ctypes.c_int64()
    _lib.check(lib.itsk_qr_workspace(d, n, ctypes.byref(nb)))
    g0 = torch.Generator(device=dev).manual_seed(d + n)
    src = torch.randn(d, n + 1, dtype=torch.float64, device=dev, generator=g0)
    ldw = n + 1 + 2
    res = []
    for rep in range(3):
        gW, W = padded(d, n + 1, ldw, dev, PAD)
        W[:, :n + 1] = src
        gR, gz, gws = Guard(8 * n * n, dev), Guard(8 * n, dev), Guard(nb.value, dev)
        R = gR.view(torch.float64, (n, n))
        z = gz.view(torch.float64, (n,))
        _lib.check(lib.itsk_qr_aug(dv.ptr(W), d, n, ldw, dv.ptr(R), dv.ptr(z), dv.ptr(gws.payload()), nb.value,
                                   dv.stream_ptr()))
        assert all(g.ok() for g in (gW, gR, gz, gws)), (d, n)
        assert pad_intact(W, n + 1)
        assert bool(torch.isfinite(R).all()) and bool(torch.isfinite(z).all())
        res.append((R.clone(), z.clone()))
    assert all(torch.equal(r[0], res[0][0]) and torch.equal(r[1], res[0][1]) for r in res[1:])


@pytest.mark.parametrize("m,n", [(999, 7), (5000, 50), (3001, 257), (4003, 500), (2503, 1025), (1201, 2000)])
def test_fused_pass_guards(env, m, n):
    itsk, _lib, dv, dev, lib = env
    lda = n + (n & 1) + 2
    gA, A = padded(m, n, lda, dev, PAD)
    A[:, :n] = torch.randn(m, n, dtype=torch.float64, device=dev)
    b, x, rp, rt = (torch.randn(k, dtype=torch.float64, device=dev) for k in (m, n, m, m))
    nb = ctypes.c_int64()
    _lib.check(lib.itsk_pass_workspace(m, n, ctypes.byref(nb)))
    res = []
    for rep in range(3):
        gr, gc, gws = Guard(8 * m, dev), Guard(8 * (n + 8), dev), Guard(nb.value, dev)
        r_out = gr.view(torch.float64, (m,))
        cs = gc.view(torch.float64, (n + 8,))
        _lib.check(lib.itsk_fused_pass(dv.ptr(A), m, n, lda, dv.ptr(b), dv.ptr(x), dv.ptr(rp), dv.ptr(r_out),
                                       dv.ptr(rt), dv.ptr(cs), dv.ptr(gws.payload()), nb.value, dv.stream_ptr()))
        assert all(g.ok() for g in (gA, gr, gc, gws)), (m, n)
        assert pad_intact(A, n)
        assert bool(torch.isfinite(r_out).all()) and bool(torch.isfinite(cs[: n + 4]).all())
        res.append((r_out.clone(), cs[: n + 4].clone()))
    assert all(torch.equal(r[0], res[0][0]) and torch.equal(r[1], res[0][1]) for r in res[1:])


def test_trsv_and_estimates_guards(env):
    itsk, _lib, dv, dev, lib = env
    for n in (50, 200, 1500):
        R = torch.triu(torch.randn(n, n, dtype=torch.float64, device=dev)) + 3 * n ** 0.5 * torch.eye(
            n, dtype=torch.float64, device=dev)
        c = torch.randn(n, dtype=torch.float64, device=dev)
        for trans in (0, 1):
            gy = Guard(8 * n, dev)
            y = gy.view(torch.float64, (n,))
            _lib.check(lib.itsk_trsv(dv.ptr(R), n, dv.ptr(c), dv.ptr(y), trans, dv.stream_ptr()))
            assert gy.ok() and bool(torch.isfinite(y).all())
        v0 = torch.randn(n, dtype=torch.float64, device=dev)
        ge = Guard(8, dev)
        _lib.check(lib.itsk_normest(dv.ptr(R), n, dv.ptr(v0), 8, dv.ptr(ge.payload()), None, dv.stream_ptr()))
        assert ge.ok() and float(ge.view(torch.float64, (1,))[0]) > 0
        nws = ctypes.c_int64()
        _lib.check(lib.itsk_condest_workspace(n, ctypes.byref(nws)))
        gk, gw = Guard(8, dev), Guard(8 * nws.value, dev)
        _lib.check(lib.itsk_condest_ws(dv.ptr(R), n, dv.ptr(v0), dv.ptr(gk.payload()), None, dv.ptr(gw.payload()),
                                       nws.value, dv.stream_ptr()))
        assert gk.ok() and gw.ok() and float(gk.view(torch.float64, (1,))[0]) >= 1.0


@pytest.fixture
def guarded_workspaces(env, monkeypatch):
    """The solver's workspaces (pattern, QR, loop, LSQR) as guarded garbage."""
    itsk, _lib, dv, dev, lib = env
    import paper_2311_04362_b200.device as devmod

    guards = []

    def workspace(nbytes, d):
        g = Guard(max(int(nbytes), 256), d)
        guards.append(g)
        return g.payload()

    monkeypatch.setattr(devmod, "workspace", workspace)
    itsk.release_workspaces()
    yield guards
    itsk.release_workspaces()


@pytest.mark.parametrize("residuals,use_graph,variant", [("all", True, "momentum"), ("last", True, "basic"),
                                                         ("last", False, "damped"), ("all", False, "basic")])
def test_solve_guards(env, guarded_workspaces, residuals, use_graph, variant):
    itsk, _lib, dv, dev, lib = env
    p = itsk.gen_randsvd(20000, 120, 1e8, 1e-6, 2)
    sols = []
    for rep in range(3):
        res = itsk.iterative_sketching(p.a, p.b, itsk.SolverConfig(d=2400, variant=variant), p.truth,
                                       residuals=residuals, use_graph=use_graph)
        sols.append((res.solution.copy(), res.iterations, list(res.trace.fe)))
    assert guarded_workspaces and all(g.ok() for g in guarded_workspaces)
    assert all(np.array_equal(s[0], sols[0][0]) and s[1:] == sols[0][1:] for s in sols[1:])
    assert np.isfinite(sols[0][0]).all()


def test_sparse_and_lsqr_guards(env, guarded_workspaces):
    itsk, _lib, dv, dev, lib = env
    p = itsk.gen_sparse(30000, 64, 3)
    r1 = itsk.iterative_sketching(p.a, p.b, itsk.SolverConfig(d=1920, max_iters=15, rng_seed=3))
    r2 = itsk.iterative_sketching(p.a, p.b, itsk.SolverConfig(d=1920, max_iters=15, rng_seed=3))
    assert np.array_equal(r1.solution, r2.solution)
    q = itsk.gen_randsvd(8000, 60, 1e8, 1e-6, 1)
    l1 = itsk.sketch_and_precondition(q.a, q.b, itsk.SolverConfig(d=1200, max_iters=20), q.truth)
    l2 = itsk.sketch_and_precondition(q.a, q.b, itsk.SolverConfig(d=1200, max_iters=20), q.truth)
    assert np.array_equal(l1.solution, l2.solution)
    assert guarded_workspaces and all(g.ok() for g in guarded_workspaces)


def test_peer_exchange_guards(env):
    """Two ranks of the peer exchange in one process with guarded receive
    buffers and flags (2 x world x (n+5) doubles, world uint64)."""
    itsk, _lib, dv, dev, lib = env
    from paper_2311_04362_b200.dist import PeerExchange, _shard_factor, _shard_prepare, shard_bounds
    from paper_2311_04362_b200.solvers import _assemble, _read_result

    m, n, d, world = 9001, 17, 340, 2
    p = itsk.gen_randsvd(m, n, 1e4, 1e-3, 4)
    so = torch.cuda.current_stream(dev)
    s = int(so.cuda_stream)
    cfg = itsk.SolverConfig(d=d, rng_seed=4, max_iters=8)
    ranks = []
    for r in range(world):
        r0, r1 = shard_bounds(m, world, r)
        ranks.append(_shard_prepare(p.a[r0:r1], p.b[r0:r1], cfg, m, r0, None, "last"))
    W = ranks[0][0].W.clone()
    for ws, *_ in ranks[1:]:
        W += ws.W
    for ws, *_ in ranks:
        ws.W.copy_(W)
    guards = [(Guard(8 * 2 * world * (n + 5), dev, fill=0), Guard(8 * world, dev, fill=0)) for _ in range(world)]
    recv = [g[0].payload() for g in guards]
    flags = [g[1].payload() for g in guards]
    pxs = [PeerExchange(r, world, [t.data_ptr() for t in recv], [t.data_ptr() for t in flags], keep=guards)
           for r in range(world)]
    ps = [_shard_factor(ws, at, lda, csr, cfg, None, px) for (ws, at, lda, csr), px in zip(ranks, pxs)]
    for r in range(world):
        _lib.check(lib.itsk_loop_begin_local(ctypes.byref(ps[r]), s))
    for r in range(world):
        _lib.check(lib.itsk_loop_begin_finish(ctypes.byref(ps[r]), s))
    for _ in range(cfg.max_iters):
        for r in range(world):
            _lib.check(lib.itsk_loop_step_pre(ctypes.byref(ps[r]), s))
        for r in range(world):
            _lib.check(lib.itsk_loop_step_post(ctypes.byref(ps[r]), s))
    outs = [_assemble(ws, _read_result(lib, ws, pr, so), None, cfg, at, ws.b)
            for (ws, at, lda, csr), pr in zip(ranks, ps)]
    assert all(g.ok() for pair in guards for g in pair)
    assert np.array_equal(outs[0].solution, outs[1].solution) and np.isfinite(outs[0].solution).all()

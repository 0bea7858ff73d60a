"""Small-size exercise of every kernel family of libitsk_b200.so, for
compute-sanitizer (memcheck / racecheck / synccheck / initcheck):

    compute-sanitizer --tool memcheck python scripts/sanitize_cases.py [family ...]

families: pattern sketch qr qr2level trsv estimates pass passrows loop loopgraph
deferred peer sparse lsqr.  Each runs one small case through the public
API / C ABI and checks the result loosely (the parity tests hold the bars;
this script only drives the kernels under the sanitizer)."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2311_04362_b200 as itsk  # noqa: E402
from paper_2311_04362_b200 import _lib  # noqa: E402
from paper_2311_04362_b200 import device as dv  # noqa: E402


def pattern():
    s = itsk.sparse_sign_new(300, 5000, 8, 1)
    assert s.rows.shape == (5000, 8)
    s = itsk.sparse_sign_new(40, 3000, 16, 2)  # many redraws
    assert s.rows.shape == (3000, 16)


def sketch():
    a = np.random.default_rng(0).standard_normal((6000, 70))
    s = itsk.sparse_sign_new(700, 6000, 8, 3)
    sa = s.apply_dense(a)
    assert np.isfinite(sa).all()


def qr():
    for m, n in [(300, 40), (4000, 201)]:
        a = np.random.default_rng(m).standard_normal((m, n))
        f = itsk.householder_qr_econ(a, a[:, 0])
        assert np.all(np.diag(f.r) >= 0)


def qr2level():
    a = np.random.default_rng(5).standard_normal((3000, 384))
    f = itsk.householder_qr_econ(a, a[:, 1])
    assert np.all(np.diag(f.r) >= 0)


def trsv():
    r = np.triu(np.random.default_rng(1).standard_normal((300, 300))) + 30 * np.eye(300)
    y = itsk.tri_solve_upper(r, np.ones(300))
    y2 = itsk.tri_solve_upper_transpose(r, np.ones(300))
    assert np.isfinite(y).all() and np.isfinite(y2).all()


def estimates():
    r = np.triu(np.random.default_rng(2).standard_normal((200, 200))) + 20 * np.eye(200)
    assert itsk.rand_power_norm_est(r) > 0 and itsk.cond_est(r) >= 1


def _pass(m, n, lda):
    dev = dv.current_device()
    g = torch.Generator(device=dev).manual_seed(m)
    store = torch.randn(m, lda, dtype=torch.float64, device=dev, generator=g)
    b = torch.randn(m, dtype=torch.float64, device=dev, generator=g)
    x = torch.randn(n, dtype=torch.float64, device=dev, generator=g)
    r_out = torch.empty(m, dtype=torch.float64, device=dev)
    cs = torch.empty(n + 8, dtype=torch.float64, device=dev)
    lib = dv.lib(dev)
    nb = ctypes.c_int64()
    _lib.check(lib.itsk_pass_workspace(m, n, ctypes.byref(nb)))
    ws = dv.workspace(nb.value, dev)
    _lib.check(lib.itsk_fused_pass(dv.ptr(store), m, n, lda, dv.ptr(b), dv.ptr(x), None, dv.ptr(r_out), None,
                                   dv.ptr(cs), dv.ptr(ws), ws.numel(), dv.stream_ptr()))
    torch.cuda.synchronize()
    assert torch.isfinite(cs[: n + 4]).all()


def pass_():
    _pass(5000, 50, 50)
    _pass(3001, 257, 258)
    _pass(999, 7, 7)


def passrows():
    _pass(3001, 513, 514)
    _pass(2003, 1500, 1500)


def loop():
    p = itsk.gen_randsvd(4000, 50, 1e6, 1e-6, 0)
    res = itsk.iterative_sketching(p.a, p.b, itsk.SolverConfig(d=1000, max_iters=8), p.truth, use_graph=False,
                                   residuals="last")
    assert res.iterations >= 1


def loopgraph():
    p = itsk.gen_randsvd(4000, 50, 1e6, 1e-6, 0)
    res = itsk.iterative_sketching(p.a, p.b, itsk.SolverConfig(d=1000, max_iters=8, variant="momentum"), p.truth,
                                   residuals="last")
    assert res.iterations >= 1


def deferred():
    p = itsk.gen_randsvd(4000, 50, 1e6, 1e-6, 0)
    res = itsk.iterative_sketching(p.a, p.b, itsk.SolverConfig(d=1000, max_iters=10), p.truth, residuals="all")
    assert res.iterations >= 1


def peer():
    """Two ranks of the peer exchange in one process (tests/test_gpu_dist.py)."""
    from paper_2311_04362_b200.dist import PeerExchange, _shard_factor, _shard_prepare, shard_bounds

    m, n, d, world = 9001, 17, 340, 2
    p = itsk.gen_randsvd(m, n, 1e4, 1e-3, 4)
    dev = dv.current_device()
    lib = dv.lib(dev)
    s = dv.stream_ptr()
    cfg = itsk.SolverConfig(d=d, rng_seed=4, max_iters=6)
    ranks = []
    for r in range(world):
        r0, r1 = shard_bounds(m, world, r)
        ranks.append(_shard_prepare(p.a[r0:r1], p.b[r0:r1], cfg, m, r0, None, "last"))
    W = ranks[0][0].W.clone()
    for ws, *_ in ranks[1:]:
        W += ws.W
    for ws, *_ in ranks:
        ws.W.copy_(W)
    bufs = [PeerExchange.buffers(n, world, dev) for _ in range(world)]
    pxs = [PeerExchange(r, world, [b[0].data_ptr() for b in bufs], [b[1].data_ptr() for b in bufs], keep=bufs)
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
    torch.cuda.synchronize()


def sparse():
    p = itsk.gen_sparse(20000, 60, 1)
    res = itsk.iterative_sketching(p.a, p.b, itsk.SolverConfig(d=1200, max_iters=6), residuals="last")
    assert res.iterations >= 1


def lsqr():
    p = itsk.gen_randsvd(4000, 50, 1e6, 1e-6, 0)
    res = itsk.sketch_and_precondition(p.a, p.b, itsk.SolverConfig(d=1000, max_iters=10), p.truth)
    assert res.iterations >= 1


FAMILIES = {"pattern": pattern, "sketch": sketch, "qr": qr, "qr2level": qr2level, "trsv": trsv,
            "estimates": estimates, "pass": pass_, "passrows": passrows, "loop": loop, "loopgraph": loopgraph,
            "deferred": deferred, "peer": peer, "sparse": sparse, "lsqr": lsqr}

if __name__ == "__main__":
    names = sys.argv[1:] or list(FAMILIES)
    torch.cuda.set_device(0)
    for nm in names:
        FAMILIES[nm]()
        torch.cuda.synchronize()
        print(f"sanitize case {nm}: ok", flush=True)

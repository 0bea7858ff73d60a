"""The row-sharded solve (dist.py) on the GPU through a real NCCL process
group.  Only one B200 exists in this environment, so the group has one rank:
the allreduces are identities and the sharded path (pattern CSR of the rank's
block, sketch + allreduce, step-wise loop around the per-iteration
allreduce, `done` polling) must reproduce the single-GPU solve bit for bit.
The multi-rank host logic is covered with gloo (test_dist_gloo.py)."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nccl_group():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import torch.distributed as dist

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield dist
    dist.destroy_process_group()


@pytest.mark.parametrize("peer", ["nccl", "auto"])
@pytest.mark.parametrize("m,n,kappa,beta,d,variant", [(20000, 60, 1e8, 1e-6, 1200, "basic"),
                                                        (50000, 200, 1e10, 1e-10, 4000, "momentum"),
                                                        (3001, 17, 1e4, 1e-3, 340, "damped")])
def test_sharded_solve_matches_single_gpu(nccl_group, m, n, kappa, beta, d, variant, peer):
    """peer="auto": the per-iteration sums go through the peer-memory exchange
    (torch symmetric memory, one rank) and the loop is one CUDA graph;
    peer="nccl": NCCL allreduce between the halves of each iteration."""
    import paper_2311_04362_b200 as itsk
    from paper_2311_04362_b200.dist import iterative_sketching_sharded

    p = itsk.gen_randsvd(m, n, kappa, beta, 3)
    cfg = itsk.SolverConfig(d=d, variant=variant, rng_seed=3)
    ref = itsk.iterative_sketching(p.a, p.b, cfg, p.truth, residuals="last")
    for rep in range(2):  # the second solve reuses the exchange buffers (next epochs)
        # rep 1 keeps every residual: the estimates then run beside the loop
        got = iterative_sketching_sharded(p.a, p.b, itsk.SolverConfig(d=d, variant=variant, rng_seed=3), m, 0,
                                          p.truth, peer=peer, residuals="last" if rep == 0 else "all")
        if peer == "auto":
            assert got.peer_exchange, "symmetric memory unavailable: peer exchange not exercised"
        _same_solve(got, ref)


def test_sharded_nonfinite_input_raises(nccl_group):
    """NaN in A: the sharded solver raises the reference's ValueError too
    (every rank holds the same R), and the next clean solve is unaffected."""
    import paper_2311_04362_b200 as itsk
    from paper_2311_04362_b200.dist import iterative_sketching_sharded

    p = itsk.gen_randsvd(5000, 40, 1e4, 1e-6, 1)
    cfg = itsk.SolverConfig(d=800, rng_seed=1)
    a = p.a.copy()
    a[123, 7] = np.nan
    with pytest.raises(ValueError, match="infs or NaNs"):
        iterative_sketching_sharded(a, p.b, cfg, 5000, 0)
    got = iterative_sketching_sharded(p.a, p.b, cfg, 5000, 0, p.truth)
    _same_solve(got, itsk.iterative_sketching(p.a, p.b, cfg, p.truth, residuals="last"))


def _same_solve(got, ref):
    assert got.trace.stop_reason == ref.trace.stop_reason
    assert got.iterations == ref.iterations
    assert np.array_equal(got.solution, ref.solution)
    assert got.trace.fe == ref.trace.fe and got.trace.re == ref.trace.re
    assert got.trace.normest == ref.trace.normest and got.trace.condest == ref.trace.condest


@pytest.mark.parametrize("m,n,d,variant,world", [(30000, 60, 1200, "basic", 2), (40001, 120, 2400, "momentum", 3),
                                                  (9001, 17, 340, "damped", 2)])
def test_peer_exchange_ranks_in_one_process(m, n, d, variant, world):
    """The peer exchange's kernels for `world` ranks, all on this one GPU and
    in one process (each rank's buffers are plain device tensors, the peers'
    pointers point at the other ranks' tensors).  Kernels never wait on work
    that has not been issued yet: per iteration every rank's pass (which
    stores its partial to all ranks and raises its flags) runs before any
    rank's tail (which waits for the flags and sums in rank order).  Every
    rank must hold the same iterates, equal bit for bit to the same sharded
    solve with the per-iteration sums formed on the host in rank order."""
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import ctypes

    import paper_2311_04362_b200 as itsk
    from paper_2311_04362_b200 import _lib
    from paper_2311_04362_b200 import device as dv
    from paper_2311_04362_b200.dist import PeerExchange, _shard_factor, _shard_prepare, shard_bounds
    from paper_2311_04362_b200.solvers import _assemble, _read_result

    p = itsk.gen_randsvd(m, n, 1e8, 1e-6, 4)
    dev = dv.current_device()
    lib = dv.lib(dev)
    so = torch.cuda.current_stream(dev)
    s = int(so.cuda_stream)

    def solve(peered: bool):
        cfg = itsk.SolverConfig(d=d, variant=variant, rng_seed=4)
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
               for r in range(world)] if peered else [None] * world
        ps = [_shard_factor(ws, at, lda, csr, cfg, None, px) for (ws, at, lda, csr), px in zip(ranks, pxs)]
        cs = [ws.cs[: n + 4] for ws, *_ in ranks]

        def host_sum():
            tot = cs[0].clone()
            for c in cs[1:]:
                tot += c
            for c in cs:
                c.copy_(tot)

        for r in range(world):
            _lib.check(lib.itsk_loop_begin_local(ctypes.byref(ps[r]), s))
        if not peered:
            host_sum()
        for r in range(world):
            _lib.check(lib.itsk_loop_begin_finish(ctypes.byref(ps[r]), s))
        for _ in range(cfg.max_iters):
            for r in range(world):
                _lib.check(lib.itsk_loop_step_pre(ctypes.byref(ps[r]), s))
            if not peered:
                host_sum()
            for r in range(world):
                _lib.check(lib.itsk_loop_step_post(ctypes.byref(ps[r]), s))
        outs = []
        for (ws, at, lda, csr), pr in zip(ranks, ps):
            res = _read_result(lib, ws, pr, so)
            outs.append(_assemble(ws, res, None, cfg, at, ws.b))
        return outs

    ref = solve(False)
    got = solve(True)
    for r in range(world):
        assert np.array_equal(ref[r].solution, ref[0].solution)
        _same_solve(got[r], ref[r])
        assert got[r].trace.residual_changes == ref[r].trace.residual_changes


def test_sharded_sparse_solve_matches_single_gpu(nccl_group):
    import paper_2311_04362_b200 as itsk
    from paper_2311_04362_b200.dist import iterative_sketching_sharded

    p = itsk.gen_sparse(40000, 80, 2)
    cfg = itsk.SolverConfig(d=2400, max_iters=15, rng_seed=2)
    ref = itsk.iterative_sketching(p.a, p.b, cfg, residuals="last")
    got = iterative_sketching_sharded(p.a, p.b, itsk.SolverConfig(d=2400, max_iters=15, rng_seed=2), 40000, 0)
    assert got.trace.stop_reason == ref.trace.stop_reason and got.iterations == ref.iterations
    assert np.array_equal(got.solution, ref.solution)


@pytest.mark.parametrize("hold", [False, True])
def test_peer_exchange_deferred_estimates_agree(hold):
    """Deferred normest / condest over 2 ranks of the peer exchange (in one
    process, as above), on a consistent system that stops after 1-2
    iterations: each rank's ready flag rises at a different time (hold=True:
    rank 1's stays zero through the whole loop and is raised just before
    itsk_loop_finish).  The ready bits travel with the partials, so both ranks
    evaluate the rule at the same iteration and stop together (a rank that
    stopped alone would leave the other waiting for its flags: ADVICE r1),
    and the result equals the solve with the estimates computed first."""
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import ctypes

    import paper_2311_04362_b200 as itsk
    from paper_2311_04362_b200 import _lib
    from paper_2311_04362_b200 import device as dv
    from paper_2311_04362_b200.dist import PeerExchange, _shard_factor, _shard_prepare, shard_bounds
    from paper_2311_04362_b200.solvers import _assemble, _read_result

    m, n, d, world = 20000, 40, 800, 2
    p = itsk.gen_randsvd(m, n, 1e3, 0.0, 5)
    dev = dv.current_device()
    lib = dv.lib(dev)
    so = torch.cuda.current_stream(dev)
    s = int(so.cuda_stream)

    def solve(defer: bool):
        cfg = itsk.SolverConfig(d=d, max_iters=12, rng_seed=5)
        ranks = []
        for r in range(world):
            r0, r1 = shard_bounds(m, world, r)
            ranks.append(_shard_prepare(p.a[r0:r1], p.b[r0:r1], cfg, m, r0, None, "all"))
        W = ranks[0][0].W.clone()
        for ws, *_ in ranks[1:]:
            W += ws.W
        for ws, *_ in ranks:
            ws.W.copy_(W)
        bufs = [PeerExchange.buffers(n, world, dev) for _ in range(world)]
        pxs = [PeerExchange(r, world, [b[0].data_ptr() for b in bufs], [b[1].data_ptr() for b in bufs], keep=bufs)
               for r in range(world)]
        ps = [_shard_factor(ws, at, lda, csr, cfg, None, px, defer=defer) for (ws, at, lda, csr), px in zip(ranks, pxs)]
        held = torch.zeros(1, dtype=torch.int64, device=dev)
        if defer and hold:
            ps[1].est_ready = held.data_ptr()
        for r in range(world):
            _lib.check(lib.itsk_loop_begin_local(ctypes.byref(ps[r]), s))
        for r in range(world):
            _lib.check(lib.itsk_loop_begin_finish(ctypes.byref(ps[r]), s))
        for _ in range(cfg.max_iters):
            for r in range(world):
                _lib.check(lib.itsk_loop_step_pre(ctypes.byref(ps[r]), s))
            for r in range(world):
                _lib.check(lib.itsk_loop_step_post(ctypes.byref(ps[r]), s))
        outs = []
        for (ws, at, lda, csr), pr in zip(ranks, ps):
            if defer:
                so.wait_stream(ws.est_stream)
                held.fill_(1)
                _lib.check(lib.itsk_loop_finish(ctypes.byref(pr), s))
            res = _read_result(lib, ws, pr, so)
            outs.append(_assemble(ws, res, None, cfg, at, ws.b))
        return outs

    ref = solve(False)
    got = solve(True)
    assert ref[0].trace.stop_reason == "stopped_by_rule" and ref[0].iterations <= 3
    for r in range(world):
        _same_solve(got[r], ref[r])
        assert np.array_equal(got[r].solution, ref[0].solution)

"""Multi-process (world_size 2, gloo, CPU) test of the row-sharded solve's
host logic: shard bounds, the pattern slice each rank owns, the two sums
(sketch once, [A'r | norms] per iteration) and the loop driver
`run_sharded_loop`.  The per-rank arithmetic is stood in by the CPU oracle;
on the GPU box the same driver calls the C-ABI kernels."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2311_04362_b200.dist import run_sharded_loop, shard_bounds


def test_shard_bounds_cover_rows():
    for m in (1, 7, 100, 200000):
        for world in (1, 2, 3, 8):
            if world > m:
                continue
            spans = [shard_bounds(m, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == m
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_bounds(10, 2, 2)


def test_loop_driver_polls_and_stops():
    calls = []
    state = {"k": 0}

    def pre():
        calls.append("pre")

    def ar():
        calls.append("ar")

    def post():
        calls.append("post")
        state["k"] += 1

    n = run_sharded_loop(pre, ar, post, lambda: state["k"] >= 6, max_iters=50, check_every=4)
    assert n == 8 and calls[:3] == ["pre", "ar", "post"]
    assert run_sharded_loop(pre, ar, post, lambda: False, max_iters=3, check_every=4) == 3
    assert run_sharded_loop(pre, ar, post, lambda: False, max_iters=0) == 0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import itsketch_oracle as orc

        m, n, d, zeta, seed = 3000, 12, 200, 8, 4
        a, b, truth = orc.gen_randsvd(m, n, 1e6, 1e-5, seed)
        pat = orc.sparse_sign_pattern(d, m, zeta, seed)
        r0, r1 = shard_bounds(m, world, rank)
        # this rank's block of S's columns
        local = orc.Pattern(d, r1 - r0, zeta, pat.rows[r0:r1], pat.signs[r0:r1], pat.scale)
        sab = torch.from_numpy(orc.sketch_apply(local, np.column_stack([a[r0:r1], b[r0:r1]])))
        dist.all_reduce(sab)
        full = orc.sketch_apply(pat, np.column_stack([a, b]))
        sketch_err = float(np.abs(sab.numpy() - full).max() / np.abs(full).max())
        q, rf = orc.householder_qr_econ(sab.numpy()[:, :n])
        x = orc.tri_solve_upper(rf, q.T @ sab.numpy()[:, n])
        normest = orc.rand_power_norm_est(rf, rng_seed=seed)
        condest = orc.cond_est(rf)
        al, bl = a[r0:r1], b[r0:r1]
        st = {"x": x, "r": bl - al @ x, "iters": 0, "done": False}
        cs = torch.zeros(n + 2, dtype=torch.float64)

        def pre():
            if st["done"]:
                cs.zero_()
                return
            c = al.T @ st["r"]
            cs.copy_(torch.from_numpy(np.concatenate([c, [0.0, 0.0]])))

        def post():
            if st["done"]:
                return
            c = cs.numpy()[:n].copy()
            step = orc.tri_solve_upper(rf, orc.tri_solve_upper_transpose(rf, c))
            xn = st["x"] + step
            rn = bl - al @ xn
            sums = torch.tensor([rn @ rn, (rn - st["r"]) @ (rn - st["r"])], dtype=torch.float64)
            dist.all_reduce(sums)
            change, resn = float(np.sqrt(sums[1])), float(np.sqrt(sums[0]))
            st["x"], st["r"] = xn, rn
            st["iters"] += 1
            bound = 2.0**-53 * (normest * np.linalg.norm(xn) + 0.04 * condest * resn)
            if change <= bound or st["iters"] >= 40:
                st["done"] = True

        issued = run_sharded_loop(pre, lambda: dist.all_reduce(cs), post, lambda: st["done"], 40, 4)
        x_ref, tr = orc.iterative_sketching(a, b, orc.Config(d=d, zeta=zeta, rng_seed=seed, max_iters=40), truth)
        out[rank] = dict(sketch_err=sketch_err, x=st["x"], iters=st["iters"], issued=issued,
                         ref_iters=len(tr.iterates) - 1, x_ref=x_ref)
    finally:
        dist.destroy_process_group()


def test_two_rank_sharded_solve_gloo():
    world = 2
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    assert res[0]["sketch_err"] < 1e-14 and res[1]["sketch_err"] < 1e-14
    # replicated state: identical iterates on both ranks
    assert np.array_equal(res[0]["x"], res[1]["x"])
    assert res[0]["iters"] == res[1]["iters"] and res[0]["issued"] == res[1]["issued"]
    assert abs(res[0]["iters"] - res[0]["ref_iters"]) <= 2
    x_ref = res[0]["x_ref"]
    assert np.linalg.norm(res[0]["x"] - x_ref) <= 1e-6 * np.linalg.norm(x_ref)


def _sparse_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import itsketch_oracle as orc
        from paper_2311_04362_b200.problems import gen_sparse

        m, n, d, zeta, seed = 5000, 30, 300, 8, 6
        p = gen_sparse(m, n, seed)
        pat = orc.sparse_sign_pattern(d, m, zeta, seed)
        r0, r1 = shard_bounds(m, world, rank)
        local = orc.Pattern(d, r1 - r0, zeta, pat.rows[r0:r1], pat.signs[r0:r1], pat.scale)
        # the rank's CSR row block and its slice of S's columns (dist.py, sparse branch)
        sa = torch.from_numpy(orc.sketch_apply_sparse(local, p.a[r0:r1]))
        dist.all_reduce(sa)
        full = orc.sketch_apply_sparse(pat, p.a)
        x = np.random.default_rng(rank).standard_normal(n)
        dist.broadcast(t := torch.from_numpy(x), src=0)
        r_loc = p.b[r0:r1] - p.a[r0:r1] @ t.numpy()
        c = torch.from_numpy(p.a[r0:r1].T @ r_loc)
        dist.all_reduce(c)
        c_full = p.a.T @ (p.b - p.a @ t.numpy())
        out[rank] = dict(sk=float(np.abs(sa.numpy() - full).max() / np.abs(full).max()),
                         c=float(np.abs(c.numpy() - c_full).max() / np.abs(c_full).max()))
    finally:
        dist.destroy_process_group()


def test_two_rank_sparse_sums_gloo():
    """The sparse branch's two sums over row blocks (S·A once, A'r per
    iteration) equal the single-block results to rounding."""
    world = 2
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_sparse_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    for r in range(world):
        assert res[r]["sk"] < 1e-14 and res[r]["c"] < 1e-13


def test_peer_exchange_params_host_logic():
    """PeerExchange (dist.py): one receive buffer and flag array per rank, at
    most ITSK_MAX_PEERS ranks, and epochs that never repeat across solves —
    every rank runs the same sequence of solves, so the sequences agree."""
    import ctypes

    from paper_2311_04362_b200 import _lib
    from paper_2311_04362_b200.dist import PeerExchange

    # the ctypes mirror of itsk_peer_params: two int32, one int64, 2 x 8 pointers
    assert ctypes.sizeof(_lib.PeerParams) == 8 + 8 + 2 * 8 * _lib.MAX_PEERS
    assert "peer" in [f for f, _ in _lib.LoopParams._fields_]
    ranks = [PeerExchange(r, 3, [100, 200, 300], [10, 20, 30]) for r in range(3)]
    seqs = [[], [], []]
    for max_iters in (50, 0, 7, 50):
        for r, px in enumerate(ranks):
            pp = px.params(max_iters)
            assert pp.rank == r and pp.size == 3
            assert list(pp.recv)[:3] == [100, 200, 300] and list(pp.flags)[:3] == [10, 20, 30]
            seqs[r].append((pp.epoch_base, max_iters))
    assert seqs[0] == seqs[1] == seqs[2]
    # a loop uses epochs base .. base + max_iters; the next one starts above
    for (b0, k0), (b1, _) in zip(seqs[0], seqs[0][1:]):
        assert b0 >= 1 and b1 > b0 + k0
    with pytest.raises(ValueError):
        PeerExchange(0, 9, list(range(9)), list(range(9)))
    with pytest.raises(ValueError):
        PeerExchange(2, 2, [1, 2], [1, 2])
    with pytest.raises(ValueError):
        PeerExchange(0, 2, [1], [1, 2])

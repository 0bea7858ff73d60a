"""Row-sharded iterative sketching over several B200s (one process per GPU).

A, b (and truth.r) are split into contiguous row blocks, rank g owning rows
[r0_g, r1_g).  Exactness follows from the column structure of the two
products on the path:

    S·[A | b] = sum_g S[:, J_g] [A_g | b_g]        (one allreduce, d x (n+1))
    A'r       = sum_g A_g' r_g                      (one allreduce per iteration,
                                                     fused with the 4 norm partials)

Everything else — the QR of the reduced sketch, x0, normest/condest, the two
triangular solves, the update, the stopping rule and the divergence guard —
is replicated: every rank holds bit-identical inputs (an allreduce returns the
same bytes on every rank) and runs the same deterministic kernels, so the
iterates agree bitwise across ranks without any further exchange.

The collective is torch.distributed.all_reduce (NCCL over NVLink/NVSwitch on
the GPU box) issued on the solver's stream between itsk_loop_step_pre and
itsk_loop_step_post.  The loop driver (`run_sharded_loop`) and the shard
arithmetic are plain host logic, tested with gloo on CPU (tests/test_dist_gloo.py).
"""

from __future__ import annotations

import collections
import ctypes
import math

import numpy as np
import torch

from . import _lib
from . import device as _dev
from .embed import pcg_state
from .linalg import normest_steps, start_vector
from .problems import Truth
from .solvers import (SolverConfig, _assemble, _loop_params, _read_result, _Workspace, update_coeffs)


def shard_bounds(m: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced row block of `rank` (first m % world ranks get one more)."""
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world of size {world}")
    base, extra = divmod(m, world)
    r0 = rank * base + min(rank, extra)
    return r0, r0 + base + (1 if rank < extra else 0)


def run_sharded_loop(step_pre, allreduce_cs, step_post, is_done, max_iters: int, check_every: int = 4) -> int:
    """Drive the replicated refinement loop around its one collective.

    Every rank calls the same sequence; the device-side control makes the
    per-iteration kernels no-ops once the stopping rule / guard fired, so the
    host only polls `is_done` every `check_every` iterations (it is identical
    on all ranks, which therefore issue the same number of collectives).
    Returns the number of iterations issued."""
    issued = 0
    while issued < max_iters:
        for _ in range(min(check_every, max_iters - issued)):
            step_pre()
            allreduce_cs()
            step_post()
            issued += 1
        if is_done():
            break
    return issued


class ShardedWorkspace(_Workspace):
    """Workspace of one rank: full-size pattern (generated on every rank from
    the shared seed), local CSR, local A / b / r_true, replicated sketch and R."""

    def __init__(self, dev, m_total, m_local, n, d, zeta, max_iters, r_slots, with_truth):
        super().__init__(dev, m_local, n, d, zeta, max_iters, r_slots, with_truth)
        self.m_total = m_total
        lib = _dev.lib(dev)
        nnz_full = m_total * zeta
        self.rows_full = torch.empty(nnz_full, dtype=torch.int32, device=dev)
        self.neg_full = torch.empty(nnz_full, dtype=torch.uint8, device=dev)
        nb = ctypes.c_int64()
        _lib.check(lib.itsk_pattern_workspace(d, m_total, zeta, ctypes.byref(nb)))
        self.pat_ws = _dev.workspace(nb.value, dev)


class PeerExchange:
    """Buffers of the loop's peer-memory exchange (itsk_peer_params): every
    rank's pass stores its reduced [c | norms] partial into every rank's
    receive buffer over NVLink and raises a flag there; every rank's tail
    waits for the flags and sums the partials in rank order.  No host
    collective per iteration, so the sharded loop runs as one CUDA graph.

    recv_ptrs / flag_ptrs are the device addresses of each rank's receive
    buffer (2 x world x (n+5) float64: c, the 4 norms and the sender's
    deferred-estimate ready bit) and flags (world uint64, zero at
    start) as seen from this rank — torch symmetric memory peers on the GPU
    box, or plain tensors of one device in the single-process tests."""

    def __init__(self, rank: int, world: int, recv_ptrs, flag_ptrs, keep=()):
        if not 1 <= world <= _lib.MAX_PEERS or not 0 <= rank < world:
            raise ValueError(f"peer exchange: rank {rank} of {world} (at most {_lib.MAX_PEERS} ranks)")
        if len(recv_ptrs) != world or len(flag_ptrs) != world:
            raise ValueError("peer exchange: one receive buffer and one flag array per rank")
        self.rank, self.world = rank, world
        self.recv_ptrs, self.flag_ptrs = [int(p) for p in recv_ptrs], [int(p) for p in flag_ptrs]
        self._keep = keep  # the tensors / handles behind the pointers
        self.next_epoch = 1

    @staticmethod
    def buffers(n: int, world: int, dev) -> tuple[torch.Tensor, torch.Tensor]:
        return (torch.zeros(2 * world * (n + 5), dtype=torch.float64, device=dev),
                torch.zeros(world, dtype=torch.int64, device=dev))

    def params(self, max_iters: int) -> _lib.PeerParams:
        """Parameters of one loop; its exchanges use epochs epoch_base ..
        epoch_base + max_iters, the next loop starts above them (every rank
        runs the same sequence of solves, so the epochs agree)."""
        pp = _lib.PeerParams()
        pp.rank, pp.size = self.rank, self.world
        pp.epoch_base = self.next_epoch
        self.next_epoch += max_iters + 2
        for r in range(self.world):
            pp.recv[r] = self.recv_ptrs[r]
            pp.flags[r] = self.flag_ptrs[r]
        return pp


_PEERS: dict = {}
# the process groups behind _PEERS' keys, kept referenced: a key holds the
# group's id(), which must not be reused by a later group with other members
# (a re-initialised default group is a new object and gets its own exchange)
_PEER_GROUPS: dict = {}


def _peer_key(group, dev, n: int, world: int) -> tuple:
    import torch.distributed as tdist

    g = group if group is not None else tdist.group.WORLD
    _PEER_GROUPS[id(g)] = g
    return (id(g), dev.index, n, world)
# why the peer exchange is unavailable, per _PEERS key (reported by the
# result's `peer_fallback` and by bench.py's `loop_exchange`)
PEER_FALLBACK: dict = {}


def peer_exchange(n: int, dev, group=None, require: bool = False) -> PeerExchange | None:
    """The rank's PeerExchange for loops with n columns on `group`, set up once
    through torch symmetric memory (IPC-mapped peer buffers over NVLink); None
    when symmetric memory is unavailable (the caller falls back to NCCL and
    the reason is kept in PEER_FALLBACK).  require=True raises instead."""
    import torch.distributed as tdist

    world = tdist.get_world_size(group)
    rank = tdist.get_rank(group)
    key = _peer_key(group, dev, n, world)
    if key in _PEERS:
        if _PEERS[key] is None and require:
            raise RuntimeError(f"peer exchange unavailable: {PEER_FALLBACK.get(key)}")
        return _PEERS[key]
    if world > _lib.MAX_PEERS:
        PEER_FALLBACK[key] = f"world size {world} > {_lib.MAX_PEERS}"
        if require:
            raise RuntimeError(f"peer exchange unavailable: {PEER_FALLBACK[key]}")
        return None
    try:
        import torch.distributed._symmetric_memory as symm_mem

        g = group if group is not None else tdist.group.WORLD
        recv = symm_mem.empty(2 * world * (n + 5), dtype=torch.float64, device=dev)
        flags = symm_mem.empty(world, dtype=torch.int64, device=dev)
        recv.zero_()
        flags.zero_()
        torch.cuda.synchronize(dev)
        hr = symm_mem.rendezvous(recv, g)
        hf = symm_mem.rendezvous(flags, g)
        tdist.barrier(group=group)  # every rank's flags are zero before any rank writes
        px = PeerExchange(rank, world, list(hr.buffer_ptrs), list(hf.buffer_ptrs), keep=(recv, flags, hr, hf))
    except Exception as exc:  # noqa: BLE001 - no symmetric memory on this setup: NCCL path
        if require:
            raise
        PEER_FALLBACK[key] = f"{type(exc).__name__}: {exc}"[:300]
        px = None
    # every rank must take the same path: a rank whose setup failed while the
    # others' succeeded would wait in NCCL for ranks that wait on peer flags
    if world > 1:
        ok = torch.tensor([1 if px is not None else 0], dtype=torch.int32, device=dev)
        tdist.all_reduce(ok, op=tdist.ReduceOp.MIN, group=group)
        if int(ok.item()) == 0 and px is not None:
            PEER_FALLBACK[key] = "the peer exchange could not be set up on another rank"
            px = None
            if require:
                raise RuntimeError(f"peer exchange unavailable: {PEER_FALLBACK[key]}")
    _PEERS[key] = px
    return px


_SWS: "collections.OrderedDict[tuple, ShardedWorkspace]" = collections.OrderedDict()


def _sharded_workspace(dev, m_total, row0, m_loc, n, d, zeta, max_iters, r_slots,
                       with_truth) -> ShardedWorkspace:
    """Per-rank workspaces (buffers, the instantiated loop graph, the peer
    parameters) reused across solves of the same shape, as on one GPU."""
    key = (dev.index, m_total, row0, m_loc, n, d, zeta, max_iters, r_slots, with_truth)
    ws = _SWS.get(key)
    if ws is None:
        ws = ShardedWorkspace(dev, m_total, m_loc, n, d, zeta, max_iters, r_slots, with_truth)
        _SWS[key] = ws
        while len(_SWS) > 2:
            _SWS.popitem(last=False)[1].release()
    else:
        _SWS.move_to_end(key)
    ws.claim_residual_rows()
    return ws


def _shard_prepare(a_local, b_local, cfg: SolverConfig, m_total: int, row0: int, truth, residuals: str):
    """Per-rank setup up to the partial sketch: workspace, local A / b /
    r_true, the full pattern from the shared seed, the CSR of this rank's
    columns of S and S[:, J_g][A_g | b_g] in ws.W (still to be summed)."""
    from .sparse import as_csr_matrix, is_sparse

    m_loc, n = int(a_local.shape[0]), int(a_local.shape[1])
    cfg.validate(n)
    if cfg.track_be:
        raise ValueError("track_be is not supported by the sharded solver")
    dev = _dev.current_device()
    lib = _dev.lib(dev)
    r_slots = cfg.max_iters + 1 if residuals == "all" else 2
    ws = _sharded_workspace(dev, m_total, row0, m_loc, n, cfg.d, cfg.zeta, cfg.max_iters, r_slots,
                            truth is not None)
    csr = None
    if is_sparse(a_local):  # a row block of a sparse A (solvers.py:195-196)
        csr = as_csr_matrix(a_local, dev)
        at, lda = None, 0
    else:
        at, lda = _dev.as_device_matrix(a_local, dev)
    ws.b.copy_(_dev.as_device_vector(b_local, dev))
    if truth is not None:
        ws.x_true.copy_(_dev.as_device_vector(truth.x, dev))
        if truth.beta > 0:
            r = truth.r
            r = r[row0:row0 + m_loc] if r.shape[0] == m_total else r
            ws.r_true.copy_(_dev.as_device_vector(r, dev))
    stream = _dev.stream_ptr()
    words, has32, pend = pcg_state(cfg.rng_seed)
    _lib.check(lib.itsk_sparse_sign_pattern(
        cfg.d, m_total, cfg.zeta, words, has32, pend, _dev.ptr(ws.rows_full), _dev.ptr(ws.neg_full),
        None, None, _dev.ptr(ws.pat_ws), ws.pat_ws.numel(), stream))
    off = row0 * cfg.zeta
    _lib.check(lib.itsk_pattern_csr(
        _dev.ptr(ws.rows_full) + 4 * off, _dev.ptr(ws.neg_full) + off, m_loc, cfg.zeta, cfg.d,
        _dev.ptr(ws.sk_ptr), _dev.ptr(ws.sk_src), _dev.ptr(ws.pat_ws), ws.pat_ws.numel(), stream))
    if csr is not None:
        _lib.check(lib.itsk_csr_sketch(csr.plan, _dev.ptr(ws.b), _dev.ptr(ws.sk_ptr), _dev.ptr(ws.sk_src), cfg.d,
                                       cfg.zeta, _dev.ptr(ws.W), ws.ldw, stream))
    else:
        _lib.check(lib.itsk_sketch(_dev.ptr(at), m_loc, n, lda, _dev.ptr(ws.b), _dev.ptr(ws.sk_ptr),
                                   _dev.ptr(ws.sk_src), cfg.d, cfg.zeta, _dev.ptr(ws.W), ws.ldw, stream))
    return ws, at, lda, csr


def _shard_factor(ws, at, lda, csr, cfg: SolverConfig, truth, peer: PeerExchange | None = None,
                  defer: bool = False):
    """Replicated part after the summed sketch: QR, x0, normest, condest and
    the loop parameters (with the peer exchange when given).  defer: the
    estimates run beside the loop (itsk_loop_params.est_ready); the caller
    joins ws.est_stream and calls itsk_loop_finish after the loop."""
    lib = _dev.lib(ws.dev)
    n = ws.n
    stream = _dev.stream_ptr()
    _lib.check(lib.itsk_qr_aug(_dev.ptr(ws.W), cfg.d, n, ws.ldw, _dev.ptr(ws.R), _dev.ptr(ws.z),
                               _dev.ptr(ws.qr_ws), ws.qr_ws.numel(), stream))
    # a non-finite R or Q'Sb (NaN / Inf in A or b): the reference's triangular
    # solve refuses it (linalg.py:59-62); R is the same on every rank, so every
    # rank raises (itsk_qr_aug has synchronised already)
    if not bool(torch.isfinite(ws.R).all() & torch.isfinite(ws.z).all()):
        from .solvers import NONFINITE_MSG

        raise ValueError(NONFINITE_MSG)
    _lib.check(lib.itsk_pack_upper(_dev.ptr(ws.R), n, _dev.ptr(ws.Rp), stream))
    if cfg.init == "zero":
        ws.xs[0].zero_()
    else:
        _lib.check(lib.itsk_trsv_rp(_dev.ptr(ws.R), _dev.ptr(ws.Rp), n, _dev.ptr(ws.z), _dev.ptr(ws.xs[0]), 0,
                                    stream))
    ws.v0.copy_(torch.from_numpy(start_vector(n, cfg.rng_seed)))
    est = _dev.ptr(ws.est)
    if defer:
        # normest / condest beside the loop's first iterations, as on one GPU
        # (solvers._sketch_qr_x0): the ready flag is raised after both
        compute = torch.cuda.current_stream(ws.dev)
        if ws.est_stream is None:
            ws.est_stream = torch.cuda.Stream(ws.dev)
            ws.est_stream2 = torch.cuda.Stream(ws.dev)
        _lib.check(lib.itsk_flag_store(est + 16, 0, stream))
        ws.est_stream.wait_stream(compute)
        ws.est_stream2.wait_stream(compute)
        _lib.check(lib.itsk_condest(_dev.ptr(ws.R), n, _dev.ptr(ws.v0), est + 8, _dev.ptr(ws.Rp),
                                    int(ws.est_stream.cuda_stream)))
        _lib.check(lib.itsk_normest(_dev.ptr(ws.R), n, _dev.ptr(ws.v0), normest_steps(n), est, _dev.ptr(ws.Rp),
                                    int(ws.est_stream2.cuda_stream)))
        ws.est_stream.wait_stream(ws.est_stream2)
        _lib.check(lib.itsk_flag_store(est + 16, 1, int(ws.est_stream.cuda_stream)))
    else:
        _lib.check(lib.itsk_normest(_dev.ptr(ws.R), n, _dev.ptr(ws.v0), normest_steps(n), est, _dev.ptr(ws.Rp),
                                    stream))
        _lib.check(lib.itsk_condest(_dev.ptr(ws.R), n, _dev.ptr(ws.v0), est + 8, _dev.ptr(ws.Rp), stream))
    alpha, beta = update_coeffs(cfg, n)
    p = _loop_params(ws, at, lda, cfg, alpha, beta, truth, m_local=ws.m, csr=csr, defer=defer)
    if peer is not None:
        # one PeerParams per workspace, updated in place: its address is part
        # of the cached graph's key, the epoch base is read on the device
        pp = peer.params(cfg.max_iters)
        if getattr(ws, "peer_params", None) is None:
            ws.peer_params = pp
        else:
            ctypes.memmove(ctypes.addressof(ws.peer_params), ctypes.addressof(pp), ctypes.sizeof(pp))
        p.peer = ctypes.addressof(ws.peer_params)
    return p


def iterative_sketching_sharded(a_local, b_local, cfg: SolverConfig, m_total: int, row0: int,
                                truth: Truth | None = None, group=None, *, residuals: str = "last",
                                check_every: int = 4, peer: str = "auto"):
    """Row-sharded solve.  Each rank passes its own block [row0, row0+m_local)
    of A and b (numpy or CUDA tensors); `truth.r` may be the full vector or
    the local slice.  A sparse block (scipy sparse / CsrMatrix) runs the CSR
    pass of sparse.cu on the rank's rows.  Returns a SolveResult whose iterates / solution / trace
    scalars are identical on every rank; residual_vectors hold the local rows.

    peer: "auto" sums the loop's per-iteration partials through the
    peer-memory exchange (PeerExchange: the pass stores to every rank over
    NVLink, the tail gathers; the whole loop is one CUDA graph) when
    symmetric memory is available and A is dense, else with NCCL allreduce
    between the two halves of each iteration (the result's `peer_fallback`
    says why); "nccl" forces the latter; "require" raises instead of falling
    back."""
    import torch.distributed as tdist

    if peer not in ("auto", "nccl", "require"):
        raise ValueError("peer must be 'auto', 'nccl' or 'require'")
    ws, at, lda, csr = _shard_prepare(a_local, b_local, cfg, m_total, row0, truth, residuals)
    lib = _dev.lib(ws.dev)
    n = ws.n
    stream_obj = torch.cuda.current_stream(ws.dev)
    stream = int(stream_obj.cuda_stream)

    def allreduce(t: torch.Tensor):
        tdist.all_reduce(t, op=tdist.ReduceOp.SUM, group=group)

    allreduce(ws.Wbuf)  # the whole padded buffer (contiguous; the pad column is zero)
    if peer == "require" and csr is not None:
        raise ValueError("peer='require': the peer exchange carries dense loops only")
    px = peer_exchange(n, ws.dev, group, require=peer == "require") if (peer != "nccl" and csr is None) else None
    fallback = None
    if px is None:
        fallback = ("peer='nccl'" if peer == "nccl" else "sparse block" if csr is not None else
                    PEER_FALLBACK.get(_peer_key(group, ws.dev, n, tdist.get_world_size(group)), "unavailable"))
    # deferred estimates: with the peer exchange the ready bits travel with
    # the partials (every rank evaluates the rule at the same iteration); the
    # host-collective loop polls `done` between collectives, so over several
    # ranks it runs with the estimates computed first
    world = tdist.get_world_size(group)
    defer = ws.r_slots == cfg.max_iters + 1 and cfg.max_iters > 0 and (px is not None or world == 1)
    p = _shard_factor(ws, at, lda, csr, cfg, truth, px, defer=defer)
    if px is not None:
        from .solvers import run_loop

        run_loop(lib, ws, p, True, stream)
    else:
        cs = ws.cs[: n + 4]
        _lib.check(lib.itsk_loop_begin_local(ctypes.byref(p), stream))
        allreduce(cs)
        _lib.check(lib.itsk_loop_begin_finish(ctypes.byref(p), stream))
        rp = ctypes.c_void_p()
        _lib.check(lib.itsk_loop_result_ptr(ctypes.byref(p), ctypes.byref(rp)))
        res_off = rp.value - _dev.ptr(ws.loop_ws)
        done_dev = ws.loop_ws[res_off + 8: res_off + 12]  # itsk_loop_result.done

        def is_done() -> bool:
            return bool(done_dev.view(torch.int32).item())

        run_sharded_loop(
            lambda: _lib.check(lib.itsk_loop_step_pre(ctypes.byref(p), stream)),
            lambda: allreduce(cs),
            lambda: _lib.check(lib.itsk_loop_step_post(ctypes.byref(p), stream)),
            is_done, cfg.max_iters, check_every)
    if defer:
        stream_obj.wait_stream(ws.est_stream)
        _lib.check(lib.itsk_loop_finish(ctypes.byref(p), stream))
    res = _read_result(lib, ws, p, stream_obj)
    out = _assemble(ws, res, truth, cfg, at, ws.b)
    out._workspace = ws  # keep the local residual rows alive
    out._csr = csr       # and the local CSR plan the trace's residuals came from
    out.peer_exchange = px is not None
    out.peer_fallback = fallback  # None, or why the loop's sums went through NCCL
    return out

"""Iterative sketching on the B200 (mirrors itsketch.solvers for the north-star path).

Drop-in for `iterative_sketching(a, b, cfg, truth)` at
/root/reference/pkg/src/itsketch/solvers.py:323-345: same SolverConfig fields
and validation, same SolveTrace / SolveResult fields, same stop reasons, same
exceptions.  Every arithmetic step runs in libitsk_b200.so on the device:

  sparse_sign_new      embed.py:83-99     device PCG64 stream (bit-identical pattern)
  S·[A | b]            embed.py:62-74     gather kernel (bit-identical to scipy)
  QR + Q'Sb, x0        solvers.py:199-210 cooperative blocked Householder, TRSV
  normest / condest    solvers.py:336-337 device power method / Lanczos
  _run_refinement      solvers.py:270-320 fused pass + TRSV pair + update + control,
                                          one CUDA graph (conditional WHILE node)

Inputs may be numpy arrays (copied to the device; pinned host memory copies
asynchronously) or CUDA fp64 tensors (used in place, zero copy).
"""

from __future__ import annotations

import collections
import ctypes
import math
import weakref
from collections.abc import Sequence
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from . import device as _dev
from .embed import default_distortion, pcg_state, SparseSignEmbedding
from .linalg import SingularMatrixError, normest_steps, start_vector
from .problems import Truth
from .sparse import as_csr_matrix, is_sparse

__all__ = ["SolverConfig", "SolveTrace", "SolveResult", "iterative_sketching", "sketch_and_solve",
           "damping_params", "momentum_params", "should_stop", "SingularMatrixError",
           "release_workspaces"]


@dataclass
class SolverConfig:
    """Field-identical to itsketch.solvers.SolverConfig (solvers.py:34-61)."""

    d: int
    zeta: int = 8
    variant: str = "basic"  # basic | damped | momentum
    init: str = "sketch_and_solve"  # sketch_and_solve | zero
    max_iters: int = 50
    unit_roundoff: float = 2.0 ** -53
    stop_gamma: float = 1.0
    stop_rho: float = 0.04
    epsilon_for_params: float | None = None  # defaults to sqrt(n/d)
    rng_seed: int = 0
    extra_iters: int = 0
    track_be: bool = False

    def validate(self, n: int) -> None:
        if self.d < n:
            raise ValueError(f"embedding dimension d={self.d} must be >= n={n}")
        if self.zeta < 1:
            raise ValueError("zeta must be >= 1")
        if self.max_iters < 0:
            raise ValueError("max_iters must be >= 0")
        if not 0 < self.unit_roundoff < 1:
            raise ValueError("unit_roundoff must be in (0, 1)")
        if self.variant not in ("basic", "damped", "momentum"):
            raise ValueError(f"unknown variant {self.variant!r}")
        if self.init not in ("sketch_and_solve", "zero"):
            raise ValueError(f"unknown init {self.init!r}")


class DeviceResiduals(Sequence):
    """SolveTrace.residual_vectors: the residual r_i of every recorded iterate,
    kept on the device and copied to numpy on first access (the reference
    keeps every m-vector; at C4 that is 32 MB per iteration)."""

    def __init__(self, rows: torch.Tensor, count: int, slots: int, first: int):
        self._rows = rows
        self._count = count
        self._base = 0  # row of index i is (i - base) % mod
        self._mod = slots
        self._first = first  # lowest index still held
        self._host: dict[int, np.ndarray] = {}

    def __len__(self) -> int:
        return self._count

    def _slot(self, i: int) -> int:
        if i < self._first:
            raise IndexError(f"residual {i} was not kept (solve ran with residuals='last')")
        return (i - self._base) % self._mod

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self[k] for k in range(*i.indices(self._count))]
        if i < 0:
            i += self._count
        if not 0 <= i < self._count:
            raise IndexError(i)
        if i not in self._host:
            self._host[i] = _dev.to_numpy(self._rows[self._slot(i)])
        return self._host[i]

    def device(self, i: int) -> torch.Tensor:
        if i < 0:
            i += self._count
        return self._rows[self._slot(i)]

    def _detach(self) -> None:
        """Called before the owning workspace is reused: keep a private copy
        of the rows still referenced."""
        keep = [self._slot(i) for i in range(self._first, self._count)]
        idx = torch.tensor(keep, dtype=torch.long, device=self._rows.device)
        self._rows = self._rows.index_select(0, idx)
        self._base = self._first
        self._mod = max(1, len(keep))


@dataclass
class SolveTrace:
    """Field-identical to itsketch.solvers.SolveTrace (solvers.py:64-74)."""

    iterates: list = field(default_factory=list)
    residual_vectors: Sequence = field(default_factory=list)
    residual_changes: list = field(default_factory=list)
    fe: list = field(default_factory=list)
    re: list = field(default_factory=list)
    be: list = field(default_factory=list)
    stop_reason: str = "max_iters"
    normest: float = 0.0
    condest: float = 0.0


@dataclass
class SolveResult:
    """solvers.py:77-85."""

    solution: np.ndarray
    trace: SolveTrace
    config: SolverConfig

    @property
    def iterations(self) -> int:
        return len(self.trace.iterates) - 1


def damping_params(epsilon: float) -> tuple[float, float]:
    """alpha = (1-eps^2)^2 / (1+eps^2), beta = 0 (solvers.py:88-92)."""
    if not 0 <= epsilon < 1:
        raise ValueError(f"need 0 <= eps < 1, got {epsilon}")
    return (1 - epsilon**2) ** 2 / (1 + epsilon**2), 0.0


def momentum_params(epsilon: float) -> tuple[float, float]:
    """alpha = (1-eps^2)^2, beta = eps^2 (solvers.py:95-99)."""
    if not 0 <= epsilon < 1:
        raise ValueError(f"need 0 <= eps < 1, got {epsilon}")
    return (1 - epsilon**2) ** 2, epsilon**2


def update_coeffs(cfg: SolverConfig, n: int) -> tuple[float, float]:
    """_update_coeffs (solvers.py:259-267)."""
    if cfg.variant == "basic":
        return 1.0, 0.0
    eps = cfg.epsilon_for_params
    if eps is None:
        eps = default_distortion(n, cfg.d)
    if cfg.variant == "damped":
        return damping_params(eps)
    return momentum_params(eps)


def should_stop(r_next, r_curr, x_next, normest, condest, u, gamma=1.0, rho=0.04) -> bool:
    """Residual-change stopping rule, inclusive (solvers.py:174-192).  The
    solver evaluates the same formula on the device (loop.cu, k_control);
    this host form is the public utility of the reference API."""
    def norm(v):
        return float(torch.linalg.vector_norm(v)) if isinstance(v, torch.Tensor) else float(np.linalg.norm(v))

    diff = (r_next - r_curr)
    change = norm(diff)
    bound = u * (gamma * normest * norm(x_next) + rho * condest * norm(r_next))
    return bool(change <= bound)


# ---------------------------------------------------------------------------
# Device workspaces (buffers + the instantiated loop graph), reused across
# solves of the same shape.
# ---------------------------------------------------------------------------
class _Workspace:
    def __init__(self, dev, m, n, d, zeta, max_iters, r_slots, with_truth):
        lib = _dev.lib(dev)
        self.dev, self.m, self.n, self.d, self.zeta = dev, m, n, d, zeta
        self.max_iters, self.r_slots = max_iters, r_slots
        f64 = dict(dtype=torch.float64, device=dev)
        nnz = m * zeta
        self.rows = torch.empty(nnz, dtype=torch.int32, device=dev)
        self.neg = torch.empty(nnz, dtype=torch.uint8, device=dev)
        self.sk_ptr = torch.empty(d + 1, dtype=torch.int32, device=dev)
        self.sk_src = torch.empty(nnz, dtype=torch.int32, device=dev)
        nb = ctypes.c_int64()
        _lib.check(lib.itsk_pattern_workspace(d, m, zeta, ctypes.byref(nb)))
        self.pat_ws = _dev.workspace(nb.value, dev)
        # W = [SA | Sb] at an even leading dimension (16-byte aligned rows for
        # the QR's vector copies); the pad column stays zero
        self.ldw = (n + 2) // 2 * 2
        self.Wbuf = torch.zeros((d, self.ldw), **f64)
        self.W = self.Wbuf[:, :n + 1]
        _lib.check(lib.itsk_qr_workspace(d, n, ctypes.byref(nb)))
        self.qr_ws = _dev.workspace(nb.value, dev)
        self.R = torch.empty((n, n), **f64)
        _lib.check(lib.itsk_pack_upper_doubles(n, ctypes.byref(nb)))
        self.Rp = torch.empty(nb.value, **f64)
        self.z = torch.empty(n, **f64)
        self.v0 = torch.empty(n, **f64)
        # iterates, trace and estimates are views of one buffer: the result is
        # read back with one device-to-host copy
        K = max_iters + 1
        self.out = torch.zeros(K * n + 4 * K + 4, **f64)
        self.xs = self.out[:K * n].view(K, n)
        self.trace = self.out[K * n:K * n + 4 * K].view(4, K)
        self.est = self.out[K * n + 4 * K:K * n + 4 * K + 3]  # normest, condest, ready flag (deferred estimates)
        self.rs = torch.empty((r_slots, m), **f64)
        self.cs = torch.zeros(n + 8, **f64)
        _lib.check(lib.itsk_loop_workspace(m, n, ctypes.byref(nb)))
        self.loop_ws = _dev.workspace(nb.value, dev)
        self.b = torch.empty(m, **f64)
        self.x_true = torch.empty(n, **f64) if with_truth else None
        self.r_true = torch.empty(m, **f64) if with_truth else None
        self.A = None  # upload buffer for host A (allocated on demand)
        self.copy_stream = None  # side stream of the chunked upload
        self.est_stream = None   # side stream of condest
        self.est_stream2 = None  # side stream of normest (deferred estimates)
        self.sing = torch.zeros(1, dtype=torch.int32, device=dev)  # QR zero-pivot flag
        self.sing_host = torch.zeros(1, dtype=torch.int32, pin_memory=True)
        self.v0_host = torch.empty(n, dtype=torch.float64, pin_memory=True)
        self.v0_seed = None
        # loop params key -> (instantiated loop graph, objects whose device
        # memory it captured: kept alive so their addresses — part of the key —
        # cannot be reused by another object while the graph is cached)
        self.graphs: dict = {}
        # residual rows: a second buffer is allocated the first time a solve
        # starts while an earlier result still refers to the rows, so results
        # kept by the caller are not copied out (two alive: the older is)
        self.rs_pool = [self.rs]
        self.rs_refs = [None]
        self.last_residuals = None
        self.host_buf = torch.empty(((max_iters + 1) * n + 4 * (max_iters + 1) + 8,),
                                    dtype=torch.float64, pin_memory=True)
        self.res_host = torch.empty(8, dtype=torch.float64, pin_memory=True)

    def claim_residual_rows(self) -> None:
        """Point self.rs at a residual buffer no live result refers to."""
        cur = next(i for i, t in enumerate(self.rs_pool) if t is self.rs)
        if self.last_residuals is not None:
            self.rs_refs[cur] = self.last_residuals
            self.last_residuals = None
        for i, ref in enumerate(self.rs_refs):
            if ref is None or ref() is None:
                self.rs_refs[i] = None
                self.rs = self.rs_pool[i]
                return
        if len(self.rs_pool) < 2:
            self.rs_pool.append(torch.empty_like(self.rs_pool[0]))
            self.rs_refs.append(None)
            self.rs = self.rs_pool[-1]
            return
        old = 1 - cur  # both in use: copy out the rows of the older result
        lr = self.rs_refs[old]()
        if lr is not None:
            lr._detach()
        self.rs_refs[old] = None
        self.rs = self.rs_pool[old]

    def embedding(self, scale) -> SparseSignEmbedding:
        return SparseSignEmbedding(d=self.d, m=self.m, zeta=self.zeta, scale=scale, rows_dev=self.rows,
                                   neg_dev=self.neg, ptr_dev=self.sk_ptr, src_dev=self.sk_src)

    def release(self):
        for h, _ in self.graphs.values():
            _lib.load().itsk_loop_graph_destroy(h)
        self.graphs = {}

    def __del__(self):
        try:
            self.release()
        except Exception:
            pass


_WS: "collections.OrderedDict[tuple, _Workspace]" = collections.OrderedDict()
_WS_MAX = 2


def _workspace(dev, m, n, d, zeta, max_iters, r_slots, with_truth) -> _Workspace:
    key = (dev.index, m, n, d, zeta, max_iters, r_slots, with_truth)
    ws = _WS.get(key)
    if ws is None:
        while len(_WS) >= _WS_MAX:
            _, old = _WS.popitem(last=False)
            old.release()
        ws = _Workspace(dev, m, n, d, zeta, max_iters, r_slots, with_truth)
        _WS[key] = ws
    else:
        _WS.move_to_end(key)
    ws.claim_residual_rows()
    return ws


def release_workspaces() -> None:
    while _WS:
        _, ws = _WS.popitem()
        ws.release()


# ---------------------------------------------------------------------------
# The solve
# ---------------------------------------------------------------------------
_PIPE_MIN_BYTES = 32 << 20   # host A at least this large is uploaded in chunks
_PIPE_CHUNK_BYTES = 48 << 20


def _upload_chunks(m: int, n: int) -> list[tuple[int, int]]:
    """Row chunks of the host upload.  The sketch of the last chunk sits
    between the end of the copy and the QR, so the tail is cut finer: the last
    standard chunk is split into quarters."""
    k = max(2, min(8, -(-8 * m * n // _PIPE_CHUNK_BYTES)))
    step = -(-m // k)
    chunks = [(r0, min(m, r0 + step)) for r0 in range(0, m, step)]
    r0, r1 = chunks.pop()
    q = max(1, -(-(r1 - r0) // 4))
    chunks += [(a, min(r1, a + q)) for a in range(r0, r1, q)]
    return chunks


def _sketch_qr_x0(lib, ws: _Workspace, at, lda, bt, cfg: SolverConfig, stream: int, csr=None, upload=None,
                  defer: bool = False):
    """Pattern, S·[A|b], QR, x0, normest, condest — solvers.py:332-337
    (S·A by apply_sparse for a CSR A, solvers.py:195-196).

    upload: a host matrix still to be copied into `at` (= ws.A).  The copy
    runs on a side stream in row chunks; the pattern is drawn while the first
    chunk is in flight and each chunk is sketched as soon as it lands
    (itsk_sketch_rows continues every sum in source order, so S·[A|b] is
    bitwise the one-shot result).

    defer: normest and condest run on side streams beside the start of the
    loop instead of before it; they enter only the stopping rule, which the
    loop evaluates once the ready flag (ws.est[2]) is set, replaying the
    iterates recorded meanwhile (itsk_loop_params.est_ready).  The caller
    joins ws.est_stream and calls itsk_loop_finish after the loop."""
    m, n, d, zeta = ws.m, ws.n, ws.d, ws.zeta
    compute = torch.cuda.current_stream(ws.dev)
    if upload is not None:
        if ws.copy_stream is None:
            ws.copy_stream = torch.cuda.Stream(ws.dev)
        ws.copy_stream.wait_stream(compute)  # earlier work on this stream still reads ws.A
    # normest / condest start vector (linalg.py:96): host draw, pinned, async
    if ws.v0_seed != cfg.rng_seed:
        ws.v0_host.copy_(torch.from_numpy(start_vector(n, cfg.rng_seed)))
        ws.v0_seed = cfg.rng_seed
    ws.v0.copy_(ws.v0_host, non_blocking=True)
    events = []

    def copy_chunk(r0, r1):
        with torch.cuda.stream(ws.copy_stream):
            at[r0:r1].copy_(upload[r0:r1], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(ws.copy_stream)
        events.append(ev)

    def copy_chunk_staged(r0, r1):  # pageable host memory: through pinned staging buffers
        events.append(_dev.upload_rows_staged(at, upload, r0, r1, ws.copy_stream))

    chunks = _upload_chunks(m, n) if upload is not None else []
    # pinned host memory: every chunk copy is queued before the pattern (whose
    # redraw rounds wait on the host), so the copy engine never idles; pageable
    # memory is staged through pinned buffers by the host (which that blocks),
    # so those copies are interleaved with the sketches
    early = upload is not None and upload.is_pinned()
    if early:
        for r0, r1 in chunks:
            copy_chunk(r0, r1)
    words, has32, pend = pcg_state(cfg.rng_seed)
    _lib.check(lib.itsk_sparse_sign_pattern(
        d, m, zeta, words, has32, pend, _dev.ptr(ws.rows), _dev.ptr(ws.neg), _dev.ptr(ws.sk_ptr),
        _dev.ptr(ws.sk_src), _dev.ptr(ws.pat_ws), ws.pat_ws.numel(), stream))
    if upload is not None:
        for k, (r0, r1) in enumerate(chunks):
            if not early:
                copy_chunk_staged(r0, r1)
            compute.wait_event(events[k])
            _lib.check(lib.itsk_sketch_rows(_dev.ptr(at), m, n, lda, _dev.ptr(bt), _dev.ptr(ws.sk_ptr),
                                            _dev.ptr(ws.sk_src), d, zeta, _dev.ptr(ws.W), ws.ldw, r0, r1,
                                            1 if k else 0, stream))
    elif csr is not None:
        _lib.check(lib.itsk_csr_sketch(csr.plan, _dev.ptr(bt), _dev.ptr(ws.sk_ptr), _dev.ptr(ws.sk_src), d, zeta,
                                       _dev.ptr(ws.W), ws.ldw, stream))
    else:
        _lib.check(lib.itsk_sketch(_dev.ptr(at), m, n, lda, _dev.ptr(bt), _dev.ptr(ws.sk_ptr),
                                   _dev.ptr(ws.sk_src), d, zeta, _dev.ptr(ws.W), ws.ldw, stream))
    # no host round trip: the zero-pivot flag is read with the results
    _lib.check(lib.itsk_qr_aug_async(_dev.ptr(ws.W), d, n, ws.ldw, _dev.ptr(ws.R), _dev.ptr(ws.z),
                                     _dev.ptr(ws.qr_ws), ws.qr_ws.numel(), _dev.ptr(ws.sing), stream))
    _lib.check(lib.itsk_pack_upper(_dev.ptr(ws.R), n, _dev.ptr(ws.Rp), stream))
    # condest (a 2-CTA cluster, the longest of the three) runs beside x0 and
    # normest (one CTA each) on a side stream; deferred, both run beside the
    # loop's first iterations
    if ws.est_stream is None:
        ws.est_stream = torch.cuda.Stream(ws.dev)
    est_ptr = _dev.ptr(ws.est)
    if defer:
        if ws.est_stream2 is None:
            ws.est_stream2 = torch.cuda.Stream(ws.dev)
        _lib.check(lib.itsk_flag_store(est_ptr + 16, 0, stream))
        ws.est_stream2.wait_stream(compute)
    ws.est_stream.wait_stream(compute)
    with torch.cuda.stream(ws.est_stream):
        _lib.check(lib.itsk_condest(_dev.ptr(ws.R), n, _dev.ptr(ws.v0), est_ptr + 8, _dev.ptr(ws.Rp),
                                    int(ws.est_stream.cuda_stream)))
    if defer:
        s2 = int(ws.est_stream2.cuda_stream)
        _lib.check(lib.itsk_normest(_dev.ptr(ws.R), n, _dev.ptr(ws.v0), normest_steps(n), est_ptr,
                                    _dev.ptr(ws.Rp), s2))
        ws.est_stream.wait_stream(ws.est_stream2)
        _lib.check(lib.itsk_flag_store(est_ptr + 16, 1, int(ws.est_stream.cuda_stream)))
    if cfg.init == "zero":
        ws.xs[0].zero_()
    else:
        _lib.check(lib.itsk_trsv_rp(_dev.ptr(ws.R), _dev.ptr(ws.Rp), n, _dev.ptr(ws.z), _dev.ptr(ws.xs[0]), 0,
                                    stream))
    if not defer:
        _lib.check(lib.itsk_normest(_dev.ptr(ws.R), n, _dev.ptr(ws.v0), normest_steps(n), est_ptr,
                                    _dev.ptr(ws.Rp), stream))
        compute.wait_stream(ws.est_stream)


NONFINITE_MSG = "array must not contain infs or NaNs"  # scipy's check_finite message


def check_singular(ws: _Workspace) -> None:
    """The QR's flags (itsk_qr_aug_async) -> the exceptions tri_solve_upper
    raises in sketch_and_solve: a zero pivot is a SingularMatrixError
    (linalg.py:54-55), a non-finite R or Q'Sb — NaN / Inf in A or b — the
    ValueError of scipy's solve_triangular (linalg.py:59-62), in that order."""
    flag = int(ws.sing_host[0])
    if flag & 1:
        raise SingularMatrixError("zero diagonal entry in triangular factor")
    if flag & 2:
        raise ValueError(NONFINITE_MSG)


def _loop_params(ws: _Workspace, at, lda, cfg: SolverConfig, alpha, beta, truth, m_local=None, csr=None,
                 defer: bool = False):
    p = _lib.LoopParams()
    p.csr = csr.plan if csr is not None else None
    p.m = ws.m if m_local is None else m_local
    p.n = ws.n
    p.lda = lda
    p.max_iters = cfg.max_iters
    p.extra_iters = cfg.extra_iters
    p.variant = 0 if cfg.variant == "basic" else 1
    p.r_slots = ws.r_slots
    p.alpha, p.beta = float(alpha), float(beta)
    p.u, p.gamma, p.rho = float(cfg.unit_roundoff), float(cfg.stop_gamma), float(cfg.stop_rho)
    p.has_truth = 1 if truth is not None else 0
    p.truth_beta = float(truth.beta) if truth is not None else 0.0
    p.A = _dev.ptr(at) if csr is None else None
    p.b = _dev.ptr(ws.b)
    p.R = _dev.ptr(ws.R)
    p.Rp = _dev.ptr(ws.Rp)
    p.x_true = _dev.ptr(ws.x_true) if truth is not None else None
    p.r_true = _dev.ptr(ws.r_true) if (truth is not None and truth.beta > 0) else None
    p.normest = _dev.ptr(ws.est)
    p.condest = _dev.ptr(ws.est) + 8
    p.xs = _dev.ptr(ws.xs)
    p.rs = _dev.ptr(ws.rs)
    p.trace = _dev.ptr(ws.trace)
    p.cs = _dev.ptr(ws.cs)
    p.ws = _dev.ptr(ws.loop_ws)
    p.ws_bytes = ws.loop_ws.numel()
    p.est_ready = _dev.ptr(ws.est) + 16 if defer else None
    # the pass's last reduction level in the tail: only without a host
    # collective between the two halves of an iteration (not the NCCL path)
    p.opts = _lib.LOOP_TAIL_SUMS if m_local is None else 0
    return p


def _params_key(p) -> tuple:
    return tuple(getattr(p, f) for f, _ in p._fields_ if f not in ("alpha", "beta", "u", "gamma", "rho",
                                                                   "truth_beta", "extra_iters"))


def _read_result(lib, ws: _Workspace, p, stream_obj) -> _lib.LoopResult:
    rp = ctypes.c_void_p()
    _lib.check(lib.itsk_loop_result_ptr(ctypes.byref(p), ctypes.byref(rp)))
    off = rp.value - _dev.ptr(ws.loop_ws)
    raw = ws.loop_ws[off:off + ctypes.sizeof(_lib.LoopResult)]
    host = ws.res_host.view(torch.uint8)[:ctypes.sizeof(_lib.LoopResult)]
    host.copy_(raw, non_blocking=True)
    ws.host_buf[:ws.out.numel()].copy_(ws.out, non_blocking=True)  # iterates, trace, estimates
    ws.sing_host.copy_(ws.sing, non_blocking=True)
    stream_obj.synchronize()
    check_singular(ws)
    return _lib.LoopResult.from_buffer_copy(bytes(host.numpy()))


def run_loop(lib, ws: _Workspace, p, use_graph: bool, stream: int, keep=None) -> None:
    """keep: the objects owning device memory the loop reads through
    pointers in `p` that are not the workspace's own (a sparse A's CSR plan):
    a cached graph holds them, so a later object cannot reuse their
    addresses and hit a graph that captured freed memory."""
    _lib.check(lib.itsk_loop_begin(ctypes.byref(p), stream))
    if p.max_iters == 0:
        return
    if use_graph:
        key = _params_key(p)
        ent = ws.graphs.get(key)
        if ent is None:
            if len(ws.graphs) >= 4:
                for g, _ in ws.graphs.values():
                    lib.itsk_loop_graph_destroy(g)
                ws.graphs = {}
            h = ctypes.c_void_p()
            _lib.check(lib.itsk_loop_graph_create(ctypes.byref(p), stream, ctypes.byref(h)))
            ent = (h, keep)
            ws.graphs[key] = ent
        _lib.check(lib.itsk_loop_graph_launch(ent[0], stream))
    else:
        for _ in range(p.max_iters):
            _lib.check(lib.itsk_loop_step_pre(ctypes.byref(p), stream))
            _lib.check(lib.itsk_loop_step_post(ctypes.byref(p), stream))


def _assemble(ws: _Workspace, res: _lib.LoopResult, truth, cfg, at, bt) -> SolveResult:
    n, K = ws.n, ws.max_iters + 1
    iters = int(res.iterations)
    hb = ws.host_buf.numpy()
    nxs = K * n
    xs = hb[:nxs].reshape(K, n)
    tr = hb[nxs:nxs + 4 * K].reshape(4, K)
    normest, condest = float(hb[nxs + 4 * K]), float(hb[nxs + 4 * K + 1])
    count = iters + 1
    trace = SolveTrace(normest=normest, condest=condest)
    trace.iterates = [xs[i].copy() for i in range(count)]
    trace.residual_changes = [float(v) for v in tr[2, :iters]]
    if truth is not None:
        trace.fe = [float(v) for v in tr[0, :count]]
        trace.re = [float(v) for v in tr[1, :count]]
    first = 0 if ws.r_slots >= count else max(0, count - ws.r_slots)
    resid = DeviceResiduals(ws.rs, count, ws.r_slots, first)
    trace.residual_vectors = resid
    ws.last_residuals = weakref.ref(resid)
    trace.stop_reason = _lib.STOP_REASONS[int(res.stop_reason)]
    if cfg.track_be:
        from .metrics import backward_error_device

        trace.be = [backward_error_device(at, bt, ws.xs[i]) for i in range(count)]
    return SolveResult(solution=trace.iterates[-1], trace=trace, config=cfg)


def iterative_sketching(a, b, cfg: SolverConfig, truth: Truth | None = None, *,
                        residuals: str = "all", use_graph: bool = True) -> SolveResult:
    """Iterative sketching (solvers.py:323-345) on the B200.

    residuals: "all" keeps every residual vector on the device (as the
    reference's trace does, copied lazily); "last" keeps only the last two
    (r_i and r_{i-1}), which bounds device memory at large m.
    """
    m, n = (a.shape if hasattr(a, "shape") else np.asarray(a).shape)
    cfg.validate(n)
    alpha, beta = update_coeffs(cfg, n)
    if residuals not in ("all", "last"):
        raise ValueError("residuals must be 'all' or 'last'")
    dev = _dev.current_device()
    lib = _dev.lib(dev)
    if cfg.track_be and m > 4000:
        raise ValueError(f"backward_error capped at m <= 4000, got m = {m}")
    r_slots = cfg.max_iters + 1 if residuals == "all" else 2
    ws = _workspace(dev, m, n, cfg.d, cfg.zeta, cfg.max_iters, r_slots, truth is not None)
    csr = None
    upload = None
    if is_sparse(a):
        # sparse A (solvers.py:195-196; section 3.5): CSR pass + CSC copy
        if cfg.track_be:
            raise ValueError("track_be is not supported for a sparse A on the B200 path")
        csr = as_csr_matrix(a, dev)
        at, lda = None, 0
    elif isinstance(a, torch.Tensor) and a.is_cuda:
        at, lda = _dev.as_device_matrix(a, dev)
    else:
        arr = np.asarray(a, dtype=np.float64)
        if ws.A is None:
            ws.A = torch.empty((m, n), dtype=torch.float64, device=dev)
        host_a = torch.from_numpy(np.ascontiguousarray(arr))
        if 8 * m * n >= _PIPE_MIN_BYTES:
            upload = host_a  # copied chunk by chunk under the pattern and the sketch
        else:
            ws.A.copy_(host_a, non_blocking=True)
        at, lda = ws.A, n
    bsrc = b if isinstance(b, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(np.asarray(b, dtype=np.float64)))
    if bsrc.shape[0] != m:
        raise ValueError(f"b has {bsrc.shape[0]} entries, A has {m} rows")
    if (bsrc.is_cuda and bsrc.device == dev and bsrc.dtype == torch.float64 and bsrc.dim() == 1
            and bsrc.is_contiguous()):
        bt = bsrc  # read in place, like A (the solver never writes b)
    else:
        ws.b.copy_(bsrc, non_blocking=True)
        bt = ws.b
    if truth is not None:
        ws.x_true.copy_(_dev.as_device_vector(truth.x, dev))
        if truth.beta > 0:
            ws.r_true.copy_(_dev.as_device_vector(truth.r, dev))
    stream_obj = torch.cuda.current_stream(dev)
    stream = int(stream_obj.cuda_stream)
    # estimates beside the loop (needs every residual kept: the stop may move
    # back to an iterate recorded before they were ready)
    defer = ws.r_slots == cfg.max_iters + 1 and cfg.max_iters > 0
    _sketch_qr_x0(lib, ws, at, lda, bt, cfg, stream, csr, upload, defer=defer)
    p = _loop_params(ws, at, lda, cfg, alpha, beta, truth, csr=csr, defer=defer)
    p.b = _dev.ptr(bt)
    run_loop(lib, ws, p, use_graph, stream, keep=csr)
    if defer:
        stream_obj.wait_stream(ws.est_stream)
        _lib.check(lib.itsk_loop_finish(ctypes.byref(p), stream))
    res = _read_result(lib, ws, p, stream_obj)
    return _assemble(ws, res, truth, cfg, at, bt)


def sketch_and_solve(a, b, s: SparseSignEmbedding):
    """Sketch-and-solve start (solvers.py:199-210): x0 = R^-1 (Q'Sb)[:n] with
    R from the QR of S·A.  Returns (x0, QrFactors(r, z)); the factors' Q (of
    S·A, linalg.py:42) is formed only if `.q` is read."""
    from .linalg import QrFactors, qr_aug, qr_row_blocks

    host = not isinstance(a, torch.Tensor)
    dev = s.rows_dev.device
    at, lda = _dev.as_device_matrix(a, dev)
    m, n = at.shape
    bt = _dev.as_device_vector(b, dev)
    w = s.apply_dense(at, bt)
    sa = w[:, :n].clone()  # S·A before the QR overwrites it (the sign reference of QrFactors.q)
    r, z = qr_aug(w, n)
    if qr_row_blocks(w.shape[0], n, dev) > 1:
        w = sa = None  # row-blocked QR: no single set of reflectors to form Q from
    if not bool(torch.isfinite(r).all() & torch.isfinite(z).all()):
        raise ValueError(NONFINITE_MSG)  # tri_solve_upper's check_finite (linalg.py:59-62)
    x0 = torch.empty(n, dtype=torch.float64, device=dev)
    _lib.check(_dev.lib(dev).itsk_trsv(_dev.ptr(r), n, _dev.ptr(z), _dev.ptr(x0), 0, _dev.stream_ptr()))
    if host:
        return _dev.to_numpy(x0), QrFactors(r=_dev.to_numpy(r), z=_dev.to_numpy(z), _v=w, _a=sa, _host=True)
    return x0, QrFactors(r=r, z=z, _v=w, _a=sa)

"""Sketch-and-precondition with LSQR on the B200 path.

Mirrors ``itsketch.solvers.lsqr`` and ``itsketch.solvers.sketch_and_precondition``
(/root/reference/pkg/src/itsketch/solvers.py:411-482, 485-525): Golub-Kahan
bidiagonalisation of A R^-1 with the Paige-Saunders recurrences and no
reorthogonalisation, started from the sketch-and-solve (or zero) iterate.

Division of labour:
  device   the m-sized work.  One bidiagonalisation step
               beta' u' = A (R^-1 v) - alpha u,   A' (beta' u')
           is ONE fused pass over A (itsk_fused_pass_scaled with b = beta u,
           bscale = -alpha/beta, x = -R^-1 v): u is kept unnormalised, so no
           extra m-vector sweep is needed.  The traced residual
           r_k = b - A x_k of every iterate is a second fused pass (the
           reference's callback does the same), which also yields
           ||r_k - r_{k-1}|| and ||r_k - r*||.  Triangular solves with R.
  host     the Golub-Kahan scalars and the n-vectors v, w, z, in the
           reference's numpy operation order (n doubles cross PCIe per step).

The pattern, S·[A|b], the QR, x0, normest and condest are the same device
kernels as iterative_sketching (solvers._sketch_qr_x0).
"""

from __future__ import annotations

import ctypes
import math
import weakref

import numpy as np
import torch

from . import _lib
from . import device as _dev
from .problems import Truth
from .solvers import (DeviceResiduals, SolverConfig, SolveResult, SolveTrace, _sketch_qr_x0, _workspace,
                      check_singular)


class _DeviceLs:
    """A, b and R on the device plus the fused-pass and TRSV plumbing."""

    def __init__(self, at: torch.Tensor, lda: int, bt: torch.Tensor, r_dev: torch.Tensor,
                 rp_dev: torch.Tensor | None = None):
        self.at, self.lda, self.bt, self.R, self.Rp = at, lda, bt, r_dev, rp_dev
        self.m, self.n = int(at.shape[0]), int(at.shape[1])
        self.dev = at.device
        self.lib = _dev.lib(self.dev)
        self.stream = _dev.stream_ptr()
        nb = ctypes.c_int64()
        _lib.check(self.lib.itsk_pass_workspace(self.m, self.n, ctypes.byref(nb)))
        self.pws = _dev.workspace(nb.value, self.dev)
        # counters zeroed once; every pass leaves them zero (ITSK_PASS_WS_READY)
        _lib.check(self.lib.itsk_pass_workspace_init(_dev.ptr(self.pws), self.m, self.n, self.stream))
        f64 = dict(dtype=torch.float64, device=self.dev)
        self.cs = torch.empty(self.n + 8, **f64)
        self.U = torch.empty((2, self.m), **f64)  # unnormalised u ring
        self.xd = torch.empty(self.n, **f64)
        self.vin = torch.empty(self.n, **f64)
        self.vout = torch.empty(self.n, **f64)
        self.host = torch.empty(self.n + 8, dtype=torch.float64, pin_memory=True)

    def rsolve(self, v: np.ndarray, trans: int) -> np.ndarray:
        """R^-1 v (trans = 0) or R^-T v (trans = 1) on the device."""
        self.vin.copy_(torch.from_numpy(np.ascontiguousarray(v, dtype=np.float64)))
        if self.Rp is not None:  # R staged from the packed layout (itsk_pack_upper)
            _lib.check(self.lib.itsk_trsv_rp(_dev.ptr(self.R), _dev.ptr(self.Rp), self.n, _dev.ptr(self.vin),
                                             _dev.ptr(self.vout), trans, self.stream))
        else:
            _lib.check(self.lib.itsk_trsv(_dev.ptr(self.R), self.n, _dev.ptr(self.vin), _dev.ptr(self.vout),
                                          trans, self.stream))
        return self.vout.cpu().numpy()

    def pass_(self, b_ptr: int, bscale: float, x: np.ndarray, r_out: torch.Tensor | None,
              r_prev: torch.Tensor | None = None, r_true: torch.Tensor | None = None, want_c: bool = False):
        """r = bscale * b - A x into r_out, c = A'r; returns (c or None, [||r||^2,
        ||r - r_prev||^2, ||r - r_true||^2, ||b||^2])."""
        self.xd.copy_(torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)))
        _lib.check(self.lib.itsk_fused_pass_ex(
            _dev.ptr(self.at), self.m, self.n, self.lda, b_ptr, float(bscale), _dev.ptr(self.xd),
            _dev.ptr(r_prev) if r_prev is not None else None, _dev.ptr(r_out) if r_out is not None else None,
            _dev.ptr(r_true) if r_true is not None else None, _dev.ptr(self.cs), _dev.ptr(self.pws),
            self.pws.numel(), _lib.PASS_WS_READY, self.stream))
        if want_c:
            self.host.copy_(self.cs)
            h = self.host.numpy()
            return h[: self.n].copy(), h[self.n: self.n + 4].copy()
        self.host[:4].copy_(self.cs[self.n: self.n + 4])
        return None, self.host[:4].numpy().copy()


def _lsqr_device(ops: _DeviceLs, x0: np.ndarray, max_iters: int, rtol: float, callback):
    """The Paige-Saunders loop of solvers.py:443-482 over the device operators."""
    n = ops.n
    z = np.zeros(n)
    # u = b - A x0 (kept as U = beta u), and A'U from the same pass
    c, nrm = ops.pass_(_dev.ptr(ops.bt), 1.0, x0, ops.U[0], want_c=True)
    beta = math.sqrt(nrm[0])
    if beta == 0.0:
        return x0.copy(), 0
    cur = 0  # U[cur] = beta_cur * u
    beta_cur = beta
    v = ops.rsolve(c / beta, 1)  # R^-T A' u
    alpha = float(np.linalg.norm(v))
    if alpha == 0.0:
        return x0.copy(), 0
    v = v / alpha
    w = v.copy()
    phibar, rhobar = beta, alpha
    anorm2 = alpha * alpha
    done = 0
    for _ in range(max_iters):
        y = ops.rsolve(v, 0)
        # beta' u' = A y - alpha u  with u = U[cur] / beta_cur (u = 0 after a breakdown)
        bscale = -alpha / beta_cur if beta_cur > 0.0 else 0.0
        nxt = 1 - cur
        c, nrm = ops.pass_(_dev.ptr(ops.U[cur]), bscale, -y, ops.U[nxt], want_c=True)
        beta = math.sqrt(nrm[0])
        if beta > 0:
            v = ops.rsolve(c / beta, 1) - beta * v
            alpha = float(np.linalg.norm(v))
            if alpha > 0:
                v = v / alpha
        cur, beta_cur = nxt, beta
        anorm2 += beta * beta + alpha * alpha
        rho = math.hypot(rhobar, beta)
        cs, sn = rhobar / rho, beta / rho
        theta = sn * alpha
        rhobar = -cs * alpha
        phi = cs * phibar
        phibar = sn * phibar
        z = z + (phi / rho) * w
        w = v - (theta / rho) * w
        done += 1
        if callback is not None:
            callback(z)
        normar = phibar * alpha * abs(cs)
        if phibar == 0.0 or normar <= rtol * math.sqrt(anorm2) * phibar:
            break
    return x0 + ops.rsolve(z, 0), done


def lsqr(a, b, x0, precond_r, max_iters: int, rtol: float = 1e-14, callback=None):
    """LSQR on min ||(b - A x0) - (A R^-1) z|| (solvers.py:411-482); returns
    (x0 + R^-1 z, iterations).  numpy or CUDA inputs; numpy out."""
    r_np = precond_r.detach().cpu().numpy() if isinstance(precond_r, torch.Tensor) else np.asarray(precond_r, float)
    if np.any(np.diag(r_np) == 0.0):
        raise _lib.SingularMatrixError("singular preconditioner")
    dev = _dev.current_device()
    at, lda = _dev.as_device_matrix(a, dev)
    bt = _dev.as_device_vector(b, dev)
    r_dev = precond_r if isinstance(precond_r, torch.Tensor) and precond_r.is_cuda else \
        torch.from_numpy(np.ascontiguousarray(r_np)).to(dev)
    x0 = x0.detach().cpu().numpy() if isinstance(x0, torch.Tensor) else np.asarray(x0, dtype=float)
    ops = _DeviceLs(at, lda, bt, r_dev.contiguous())
    return _lsqr_device(ops, x0, max_iters, rtol, callback)


def sketch_and_precondition(a, b, cfg: SolverConfig, truth: Truth | None = None, *,
                            residuals: str = "all") -> SolveResult:
    """Sketch, QR of the sketch, LSQR on A R^-1 from the sketch-and-solve (or
    zero) start (solvers.py:485-525).  residuals="last" keeps only the last
    two residual vectors on the device (as iterative_sketching)."""
    m, n = (a.shape if hasattr(a, "shape") else np.asarray(a).shape)
    cfg.validate(n)
    if residuals not in ("all", "last"):
        raise ValueError("residuals must be 'all' or 'last'")
    if cfg.track_be:
        raise ValueError("track_be is not supported by the B200 sketch_and_precondition")
    dev = _dev.current_device()
    lib = _dev.lib(dev)
    slots = cfg.max_iters + 1 if residuals == "all" else 2
    ws = _workspace(dev, m, n, cfg.d, cfg.zeta, cfg.max_iters, slots, truth is not None)
    at, lda = _dev.as_device_matrix(a, dev)
    ws.b.copy_(_dev.as_device_vector(b, dev))
    stream = _dev.stream_ptr()
    _sketch_qr_x0(lib, ws, at, lda, ws.b, cfg, stream)
    est = ws.est.cpu().numpy()
    ws.sing_host.copy_(ws.sing)
    check_singular(ws)
    trace = SolveTrace(normest=float(est[0]), condest=float(est[1]))
    x0 = ws.xs[0].cpu().numpy()
    r_true = None
    xt = None
    if truth is not None:
        xt = np.asarray(truth.x, dtype=float)
        if truth.beta > 0:
            ws.r_true.copy_(_dev.as_device_vector(truth.r, dev))
            r_true = ws.r_true
    ops = _DeviceLs(at, lda, ws.b, ws.R, ws.Rp)
    rs = ws.rs
    count = [0]
    bnorm = [None]

    def record(x: np.ndarray, first: bool):
        k = count[0]
        prev = None if first else rs[(k - 1) % slots]
        _, nrm = ops.pass_(_dev.ptr(ws.b), 1.0, x, rs[k % slots], r_prev=prev, r_true=r_true)
        if first:
            bnorm[0] = math.sqrt(nrm[3])
        else:
            trace.residual_changes.append(math.sqrt(nrm[1]))
        trace.iterates.append(x)
        if truth is not None:
            trace.fe.append(float(np.linalg.norm(xt - x) / np.linalg.norm(xt)))
            trace.re.append(math.sqrt(nrm[2]) / truth.beta if truth.beta > 0 else math.sqrt(nrm[0]) / bnorm[0])
        count[0] = k + 1

    record(x0, True)
    x, _ = _lsqr_device(ops, x0, cfg.max_iters, cfg.unit_roundoff,
                        lambda z: record(x0 + ops.rsolve(z, 0), False))
    trace.stop_reason = "max_iters" if len(trace.iterates) - 1 >= cfg.max_iters else "stopped_by_rule"
    # lsqr's returned x is computed exactly like the last traced iterate
    # (x0 + R^-1 z on the same device solve), so r, FE and RE of the last entry
    # already describe it (solvers.py:517-524)
    trace.iterates[-1] = x
    total = count[0]
    resid = DeviceResiduals(rs, total, slots, 0 if slots >= total else total - slots)
    trace.residual_vectors = resid
    ws.last_residuals = weakref.ref(resid)  # detached if the workspace is reused
    return SolveResult(solution=x, trace=trace, config=cfg)

"""Dense kernels on the sketch's R factor (mirrors itsketch.linalg for the path).

    householder_qr_econ  linalg.py:30-47    -> device blocked Householder QR
    tri_solve_upper      linalg.py:59-62    -> device back substitution
    tri_solve_upper_transpose linalg.py:65-68 -> device forward substitution
    rand_power_norm_est  linalg.py:79-105   -> device power method, same start vector
    cond_est             linalg.py:108-113  -> device Lanczos extremes of R'R, R^-1 R^-T

Differences from the reference, by design:
  * the QR does not form Q (dorgqr) on the solver path; it applies the
    reflectors to an extra right-hand-side column instead, returning R and
    z = Q'rhs.  QrFactors.q forms Q on first access from the Householder
    vectors (householder_qr_econ keeps them).
  * cond_est uses Lanczos (<= 96 steps, stopped when the extreme Ritz values
    are stable to rounding) instead of a full SVD; for the spectra on this
    path it agrees with dgesdd's ratio to ~1e-14 relative (tests/).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from . import device as _dev
from ._lib import SingularMatrixError

__all__ = ["QrFactors", "SingularMatrixError", "householder_qr_econ", "qr_aug", "tri_solve_upper",
           "tri_solve_upper_transpose", "rand_power_norm_est", "cond_est", "normest_steps"]


@dataclass(frozen=True)
class QrFactors:
    """R (n x n, upper, diag >= 0), z = Q' rhs (None without a rhs), and Q.

    The reference's QrFactors (linalg.py:21-27) carries an explicit Q from
    dorgqr.  The solver path never needs it (the reflectors are applied to the
    rhs column instead, solvers.py:209 only needs Q'Sb), so `q` is formed on
    first access from the Householder vectors the device QR leaves below the
    diagonal (`_form_q`; float64 GEMMs through torch, off the solver path)."""

    r: object
    z: object = None
    _v: object = field(default=None, repr=False, compare=False)   # the factored [V \ R | .] (device)
    _a: object = field(default=None, repr=False, compare=False)   # the input (device), for the sign of diag(R)
    _host: bool = field(default=False, repr=False, compare=False)

    @property
    def q(self):
        """Q (m x n, orthonormal columns, Q R = A) as linalg.py:42-46 returns it."""
        cached = self.__dict__.get("_q")
        if cached is None:
            if self._v is None:
                raise AttributeError("QrFactors.q: built without the Householder vectors (by hand, or by the "
                                     "row-blocked QR of more than ~50000 rows); householder_qr_econ(a) of a "
                                     "shorter matrix returns a QrFactors that can form Q")
            qd = _form_q(self._v, self.r.shape[0], self._a)
            cached = _dev.to_numpy(qd) if self._host else qd
            object.__setattr__(self, "_q", cached)
        return cached


def _form_q(w: torch.Tensor, n: int, a: torch.Tensor, nb: int = 128) -> torch.Tensor:
    """Q = H_1 ... H_n [I; 0] (dorgqr) from the factored matrix: column j of
    `w` holds v_j below the diagonal (unit diagonal implied).  tau_j =
    2 / v_j'v_j (dlarfg's (beta - alpha) / beta), 0 for an exactly zero tail
    (H_j = I); blocks of nb reflectors are applied last block first as
    I - V T V' with T^-1 = diag(1/tau) + striu(V'V) (dlarft).  The columns are
    then signed like R's rows (diag(R) >= 0, linalg.py:43-46)."""
    d = w.shape[0]
    dev = w.device
    q = torch.zeros((d, n), dtype=torch.float64, device=dev)
    q.diagonal().fill_(1.0)
    for k1 in range(n, 0, -nb):
        k0 = max(0, k1 - nb)
        v = torch.tril(w[k0:, k0:k1], -1)
        live = (v != 0).any(0)                 # reflectors with a non-zero tail
        v.diagonal().copy_(live.to(torch.float64))
        g = v.T @ v
        tinv = torch.triu(g, 1)
        tinv.diagonal().copy_(torch.where(live, 0.5 * g.diagonal(), torch.ones_like(g.diagonal())))
        qs = q[k0:, :]
        y = v.T @ qs
        zt = torch.linalg.solve_triangular(tinv, y, upper=True)
        qs.sub_(v @ zt)
    sgn = torch.sign((q * a).sum(0))
    sgn = torch.where(sgn == 0, torch.ones_like(sgn), sgn)
    q.mul_(sgn)
    return q


def qr_row_blocks(d: int, n: int, dev) -> int:
    """Row blocks of the device QR of a d x n matrix (itsk_qr_row_blocks)."""
    k = ctypes.c_int64()
    _lib.check(_dev.lib(dev).itsk_qr_row_blocks(d, n, ctypes.byref(k)))
    return int(k.value)


def qr_workspace(d: int, n: int, dev) -> torch.Tensor:
    lib = _dev.lib(dev)
    nbytes = ctypes.c_int64()
    _lib.check(lib.itsk_qr_workspace(d, n, ctypes.byref(nbytes)))
    return _dev.workspace(nbytes.value, dev)


def qr_aug(w: torch.Tensor, n: int, r_out: torch.Tensor | None = None, z_out: torch.Tensor | None = None,
           ws: torch.Tensor | None = None):
    """In-place Householder QR of the device matrix w = [SA | Sb] (d x (n+1),
    or d x n without a rhs).  Returns (R, z).  Raises SingularMatrixError like
    the reference's tri_solve_upper on an exactly-zero R_kk."""
    dev = w.device
    d = w.shape[0]
    has_rhs = w.shape[1] > n
    if r_out is None:
        r_out = torch.empty((n, n), dtype=torch.float64, device=dev)
    if has_rhs and z_out is None:
        z_out = torch.empty(n, dtype=torch.float64, device=dev)
    if ws is None:
        ws = qr_workspace(d, n, dev)
    lib = _dev.lib(dev)
    _lib.check(lib.itsk_qr_aug(_dev.ptr(w), d, n, int(w.stride(0)), _dev.ptr(r_out),
                               _dev.ptr(z_out) if has_rhs else None, _dev.ptr(ws), ws.numel(),
                               _dev.stream_ptr()))
    return r_out, (z_out if has_rhs else None)


def householder_qr_econ(a, rhs=None) -> QrFactors:
    """Economy QR with nonnegative diag(R) (linalg.py:30-47) on the device.
    With `rhs`, also returns z = Q' rhs (solvers.py:209)."""
    host = not isinstance(a, torch.Tensor)
    dev = _dev.current_device() if host else a.device
    at, _ = _dev.as_device_matrix(a, dev)
    d, n = at.shape
    if d < n:
        raise ValueError(f"need m >= n, got {d} x {n}")
    ncol = n + (1 if rhs is not None else 0)
    w = torch.empty((d, ncol), dtype=torch.float64, device=dev)
    w[:, :n] = at
    if rhs is not None:
        w[:, n] = _dev.as_device_vector(rhs, dev)
    r, z = qr_aug(w, n)
    # w (the Householder vectors) and the input stay on the device behind the
    # result so that .q can be formed on request — unless the factorisation
    # ran over row blocks (TSQR beyond ~50000 rows: no single set of reflectors)
    if qr_row_blocks(d, n, dev) > 1:
        w = at = None
    if host:
        return QrFactors(r=_dev.to_numpy(r), z=None if z is None else _dev.to_numpy(z), _v=w, _a=at, _host=True)
    return QrFactors(r=r, z=z, _v=w, _a=at)


def _solve(r, c, trans: int):
    host = not isinstance(r, torch.Tensor)
    dev = _dev.current_device() if host else r.device
    rt, _ = _dev.as_device_matrix(r, dev)
    n = rt.shape[0]
    if rt.shape[0] != rt.shape[1]:
        raise ValueError(f"expected a square matrix, got shape {tuple(rt.shape)}")
    if host and np.any(np.diag(np.asarray(r, dtype=float)) == 0.0):
        raise SingularMatrixError("zero diagonal entry in triangular factor")
    if not host and bool((torch.diagonal(rt) == 0).any()):
        raise SingularMatrixError("zero diagonal entry in triangular factor")
    rt = rt.contiguous()
    ct = _dev.as_device_vector(c, dev)
    if not bool(torch.isfinite(rt).all() & torch.isfinite(ct).all()):
        raise ValueError("array must not contain infs or NaNs")  # scipy solve_triangular's check_finite
    y = torch.empty(n, dtype=torch.float64, device=dev)
    _lib.check(_dev.lib(dev).itsk_trsv(_dev.ptr(rt), n, _dev.ptr(ct), _dev.ptr(y), trans, _dev.stream_ptr()))
    return _dev.to_numpy(y) if host else y


def tri_solve_upper(r, c):
    """Solve R y = c (linalg.py:59-62)."""
    return _solve(r, c, 0)


def tri_solve_upper_transpose(r, c):
    """Solve R' y = c (linalg.py:65-68)."""
    return _solve(r, c, 1)


def normest_steps(n: int, steps: int | None = None) -> int:
    if steps is None:
        steps = max(1, math.ceil(math.log2(n))) if n > 1 else 1
    if steps < 1:
        raise ValueError("steps must be >= 1")
    return steps


def start_vector(n: int, rng_seed: int) -> np.ndarray:
    """default_rng(seed).standard_normal(n) — the start vector of linalg.py:96."""
    return np.random.default_rng(rng_seed).standard_normal(n)


def _scalar_out(dev):
    return torch.empty(1, dtype=torch.float64, device=dev)


def rand_power_norm_est(r, steps: int | None = None, rng_seed: int = 0, out: torch.Tensor | None = None):
    """Randomized power estimate of ||R||_2 (linalg.py:79-105) on the device."""
    host = not isinstance(r, torch.Tensor)
    dev = _dev.current_device() if host else r.device
    rt, _ = _dev.as_device_matrix(r, dev)
    rt = rt.contiguous()
    n = rt.shape[0]
    steps = normest_steps(n, steps)
    v0 = _dev.as_device_vector(start_vector(n, rng_seed), dev)
    res = out if out is not None else _scalar_out(dev)
    _lib.check(_dev.lib(dev).itsk_normest(_dev.ptr(rt), n, _dev.ptr(v0), steps, _dev.ptr(res), None,
                                          _dev.stream_ptr()))
    return float(res.item()) if (host or out is None) else res


def cond_est(r, rng_seed: int = 0, out: torch.Tensor | None = None):
    """kappa_2(R) = sigma_max / sigma_min (linalg.py:108-113) on the device."""
    host = not isinstance(r, torch.Tensor)
    dev = _dev.current_device() if host else r.device
    rt, _ = _dev.as_device_matrix(r, dev)
    rt = rt.contiguous()
    if rt.shape[0] != rt.shape[1]:
        raise ValueError(f"expected a square matrix, got shape {tuple(rt.shape)}")
    if bool((torch.diagonal(rt) == 0).any()):
        raise SingularMatrixError("zero diagonal entry in triangular factor")
    n = rt.shape[0]
    v0 = _dev.as_device_vector(start_vector(n, rng_seed), dev)
    res = out if out is not None else _scalar_out(dev)
    nws = ctypes.c_int64()
    _lib.check(_dev.lib(dev).itsk_condest_workspace(n, ctypes.byref(nws)))
    ws = torch.empty(nws.value, dtype=torch.float64, device=dev)
    _lib.check(_dev.lib(dev).itsk_condest_ws(_dev.ptr(rt), n, _dev.ptr(v0), _dev.ptr(res), None, _dev.ptr(ws),
                                             ws.numel(), _dev.stream_ptr()))
    return float(res.item()) if (host or out is None) else res

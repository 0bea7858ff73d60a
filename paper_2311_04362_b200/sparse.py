"""Sparse CSR A on the B200.

The reference solves with a scipy sparse A on the same path: S·A through
SparseSignEmbedding.apply_sparse (embed.py:76-80, dispatched at
solvers.py:195-196) and the loop's `b - a @ x` / `a.T @ r` (solvers.py:290,
299, 343) as scipy CSR / CSC matvecs.  `CsrMatrix` uploads the CSR arrays
once and owns the library's plan (`itsk_csr_plan_create`: the CSC copy and
the chunk table of the A'r pass); `iterative_sketching` accepts a scipy
sparse matrix or a `CsrMatrix` wherever a dense A is accepted.
"""

from __future__ import annotations

import ctypes

import numpy as np
import scipy.sparse as sp
import torch

from . import _lib
from . import device as _dev


class CsrMatrix:
    """A CSR matrix resident on the device plus its pass plan.

    Built from a scipy sparse matrix (converted to CSR, values to float64;
    the stored order — duplicates included — is kept, as scipy's own
    products keep it) or from device tensors (row_ptr int64 m+1, col int32,
    val float64)."""

    def __init__(self, row_ptr: torch.Tensor, col: torch.Tensor, val: torch.Tensor, shape: tuple[int, int]):
        m, n = int(shape[0]), int(shape[1])
        if row_ptr.dtype != torch.int64 or col.dtype != torch.int32 or val.dtype != torch.float64:
            raise ValueError("CsrMatrix needs row_ptr int64, col int32, val float64")
        if row_ptr.numel() != m + 1 or col.numel() != val.numel():
            raise ValueError("CSR arrays do not match the shape")
        self.shape = (m, n)
        self.nnz = int(val.numel())
        self.row_ptr, self.col, self.val = row_ptr.contiguous(), col.contiguous(), val.contiguous()
        self.dev = row_ptr.device
        self._lib = _dev.lib(self.dev)
        h = ctypes.c_void_p()
        _lib.check(self._lib.itsk_csr_plan_create(
            _dev.ptr(self.row_ptr), _dev.ptr(self.col) if self.nnz else None, _dev.ptr(self.val) if self.nnz else None,
            m, n, self.nnz, _dev.stream_ptr(), ctypes.byref(h)))
        self.plan = h

    @classmethod
    def from_scipy(cls, a, dev: torch.device | None = None) -> "CsrMatrix":
        dev = dev if dev is not None else _dev.current_device()
        a = a if a.format == "csr" else a.tocsr()
        pin = torch.cuda.is_available()

        def up(x, dt):
            t = torch.from_numpy(np.ascontiguousarray(x, dtype=dt))
            return (t.pin_memory() if pin else t).to(dev, non_blocking=True)

        return cls(up(a.indptr, np.int64), up(a.indices, np.int32), up(a.data, np.float64), a.shape)

    def close(self) -> None:
        if getattr(self, "plan", None):
            self._lib.itsk_csr_plan_destroy(self.plan)
            self.plan = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- the pass (r = b - A x, c = A'r, norms) ------------------------------
    def pass_(self, b: torch.Tensor, x: torch.Tensor, r_out: torch.Tensor | None = None,
              r_prev: torch.Tensor | None = None, r_true: torch.Tensor | None = None,
              bscale: float = 1.0) -> torch.Tensor:
        """cs = [A'r (n) | |r|^2, |r - r_prev|^2, |r_true - r|^2, |b|^2] with
        r = bscale*b - A x (written to r_out when given)."""
        cs = torch.empty(self.shape[1] + 8, dtype=torch.float64, device=self.dev)
        _lib.check(self._lib.itsk_csr_pass(self.plan, _dev.ptr(b), float(bscale), _dev.ptr(x), _dev.ptr(r_prev),
                                           _dev.ptr(r_out), _dev.ptr(r_true), _dev.ptr(cs), _dev.stream_ptr()))
        return cs

    def sketch(self, emb, b: torch.Tensor | None, out: torch.Tensor | None = None) -> torch.Tensor:
        """S·[A | b] (d x (n+1)), or S·A without b — bitwise apply_sparse."""
        n = self.shape[1]
        ncol = n + (1 if b is not None else 0)
        if out is None:
            out = torch.empty((emb.d, ncol), dtype=torch.float64, device=self.dev)
        _lib.check(self._lib.itsk_csr_sketch(self.plan, _dev.ptr(b), _dev.ptr(emb.ptr_dev), _dev.ptr(emb.src_dev),
                                             emb.d, emb.zeta, _dev.ptr(out), int(out.stride(0)), _dev.stream_ptr()))
        return out


def as_csr_matrix(a, dev: torch.device) -> CsrMatrix:
    if isinstance(a, CsrMatrix):
        return a
    return CsrMatrix.from_scipy(a, dev)


def is_sparse(a) -> bool:
    return isinstance(a, CsrMatrix) or sp.issparse(a)


def residual_norm_device(a, b, x) -> float:
    """||b - A x|| through the device pass (sparsebench's final_resnorm,
    cli.py:271)."""
    dev = _dev.current_device()
    A = as_csr_matrix(a, dev)
    bt = _dev.as_device_vector(b, dev)
    xt = _dev.as_device_vector(x, dev)
    cs = A.pass_(bt, xt)
    return float(torch.sqrt(cs[A.shape[1]]).item())

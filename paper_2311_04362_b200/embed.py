"""Sparse sign embedding on the B200 (mirrors itsketch.embed for the path).

sparse_sign_new (embed.py:83-99) draws the pattern on the device from the
same numpy PCG64 stream as the reference (libitsk_b200 `itsk_sparse_sign_pattern`),
so `rows` / `signs` are bit-identical to the reference's, and apply_dense /
apply_vec (embed.py:62-74) run the deterministic gather kernel whose sums are
bit-identical to scipy's csc_matvecs.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from . import device as _dev


def pcg_state(rng_seed: int):
    """(state_hi, state_lo, inc_hi, inc_lo), has_uint32, uinteger of
    np.random.default_rng(rng_seed) — the stream embed.py:89 draws from."""
    st = np.random.default_rng(rng_seed).bit_generator.state
    s, inc = int(st["state"]["state"]), int(st["state"]["inc"])
    m64 = (1 << 64) - 1
    words = (ctypes.c_uint64 * 4)(s >> 64, s & m64, inc >> 64, inc & m64)
    return words, int(st["has_uint32"]), int(st["uinteger"])


@dataclass
class SparseSignEmbedding:
    """Sparse sign embedding S (d x m), zeta nonzeros +-1/sqrt(zeta) per column,
    resident on the device.

    Device layout: `rows_dev`/`neg_dev` in the reference's (m, zeta) order
    (uint32 / uint8), and the same pattern grouped by sketch row,
    `ptr_dev` (d+1) / `src_dev` (m*zeta; source row | sign<<31), sources
    ascending — the order the gather kernel sums in."""

    d: int
    m: int
    zeta: int
    scale: float
    rows_dev: torch.Tensor
    neg_dev: torch.Tensor
    ptr_dev: torch.Tensor
    src_dev: torch.Tensor
    _cache: dict = field(default_factory=dict, repr=False, compare=False)

    @property
    def rows(self) -> np.ndarray:
        """(m, zeta) int64 row indices (host copy, for inspection)."""
        if "rows" not in self._cache:
            self._cache["rows"] = _dev.to_numpy(self.rows_dev).view(np.uint32).astype(np.int64).reshape(
                self.m, self.zeta)
        return self._cache["rows"]

    @property
    def signs(self) -> np.ndarray:
        """(m, zeta) float64 +-1 (host copy)."""
        if "signs" not in self._cache:
            neg = _dev.to_numpy(self.neg_dev).reshape(self.m, self.zeta)
            self._cache["signs"] = np.where(neg != 0, -1.0, 1.0)
        return self._cache["signs"]

    @property
    def matrix(self):
        """scipy CSC view (host), as SparseSignEmbedding.matrix (embed.py:57-60)."""
        import scipy.sparse as sp

        data = (self.signs * self.scale).ravel()
        return sp.csc_matrix((data, self.rows.ravel(), self.zeta * np.arange(self.m + 1)),
                             shape=(self.d, self.m))

    def apply_dense(self, a, b=None, out: torch.Tensor | None = None):
        """S @ a for an m x n matrix or length-m vector (embed.py:62-67).
        With `b`, returns S @ [a | b] as one d x (n+1) device matrix (the
        solver's fused form).  numpy in -> numpy out; CUDA tensor in ->
        CUDA tensor out."""
        host = not isinstance(a, torch.Tensor)
        dev = self.rows_dev.device
        vec = (np.ndim(a) == 1) if host else a.ndim == 1
        if vec:
            if b is not None:
                raise ValueError("apply_dense(vector, b) is not supported")
            bt = _dev.as_device_vector(a, dev)
            if bt.shape[0] != self.m:
                raise ValueError(f"dimension mismatch: S is {self.d}x{self.m}, input has {bt.shape[0]} rows")
            res = self._sketch(None, 0, 0, bt, out)
            res = res[:, 0]
        else:
            at, lda = _dev.as_device_matrix(a, dev)
            if at.shape[0] != self.m:
                raise ValueError(f"dimension mismatch: S is {self.d}x{self.m}, input has {at.shape[0]} rows")
            bt = None if b is None else _dev.as_device_vector(b, dev)
            res = self._sketch(at, at.shape[1], lda, bt, out)
        return _dev.to_numpy(res) if host else res

    def apply_vec(self, v):
        """S @ v for a length-m vector (embed.py:69-74)."""
        if (np.ndim(v) if not isinstance(v, torch.Tensor) else v.ndim) != 1:
            raise ValueError("apply_vec expects a vector")
        return self.apply_dense(v)

    def apply_sparse(self, a, b=None):
        """S @ a for a sparse m x n matrix, dense result (embed.py:76-80) —
        bitwise scipy's (S_csc @ a.tocsc()).todense().  `a` is a scipy sparse
        matrix (numpy result) or a sparse.CsrMatrix (device result); with `b`,
        S @ [a | b]."""
        from .sparse import CsrMatrix, as_csr_matrix

        dev = self.rows_dev.device
        A = as_csr_matrix(a, dev)
        if A.shape[0] != self.m:
            raise ValueError(f"dimension mismatch: S is {self.d}x{self.m}, input has {A.shape[0]} rows")
        bt = None if b is None else _dev.as_device_vector(b, dev)
        res = A.sketch(self, bt)
        return res if isinstance(a, CsrMatrix) else _dev.to_numpy(res)

    def _sketch(self, at, n, lda, bt, out):
        dev = self.rows_dev.device
        ncol = n + (1 if bt is not None else 0)
        if out is None:
            out = torch.empty((self.d, ncol), dtype=torch.float64, device=dev)
        lib = _dev.lib(dev)
        _lib.check(lib.itsk_sketch(
            _dev.ptr(at), self.m, n, max(lda, n), _dev.ptr(bt), _dev.ptr(self.ptr_dev), _dev.ptr(self.src_dev),
            self.d, self.zeta, _dev.ptr(out), int(out.stride(0)), _dev.stream_ptr()))
        return out


def sparse_sign_new(d: int, m: int, zeta: int, rng_seed: int, device=None) -> SparseSignEmbedding:
    """Construct the sparse sign embedding of embed.py:83-99 on the device."""
    if d < 1 or m < 1:
        raise ValueError("d and m must be >= 1")
    if not 1 <= zeta <= d:
        raise ValueError(f"need 1 <= zeta <= d, got zeta={zeta}, d={d}")
    dev = torch.device(device) if device is not None else _dev.current_device()
    lib = _dev.lib(dev)
    nnz = m * zeta
    rows = torch.empty(nnz, dtype=torch.int32, device=dev)
    neg = torch.empty(nnz, dtype=torch.uint8, device=dev)
    ptr = torch.empty(d + 1, dtype=torch.int32, device=dev)
    src = torch.empty(nnz, dtype=torch.int32, device=dev)
    nbytes = ctypes.c_int64()
    _lib.check(lib.itsk_pattern_workspace(d, m, zeta, ctypes.byref(nbytes)))
    ws = _dev.workspace(nbytes.value, dev)
    words, has32, pend = pcg_state(rng_seed)
    _lib.check(lib.itsk_sparse_sign_pattern(
        d, m, zeta, words, has32, pend, _dev.ptr(rows), _dev.ptr(neg), _dev.ptr(ptr), _dev.ptr(src),
        _dev.ptr(ws), ws.numel(), _dev.stream_ptr()))
    return SparseSignEmbedding(d=d, m=m, zeta=zeta, scale=1.0 / math.sqrt(zeta), rows_dev=rows,
                               neg_dev=neg, ptr_dev=ptr, src_dev=src)


def default_distortion(n: int, d: int) -> float:
    """sqrt(n/d) (embed.py:132-135)."""
    return math.sqrt(n / d)

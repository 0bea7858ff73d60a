"""Problem instances (mirrors itsketch.problems: Truth, LsProblem, gen_randsvd).

gen_randsvd is the controlled-spectrum generator that defines every
BASELINE.json configuration (/root/reference/pkg/src/itsketch/problems.py:65-89).
It runs on the host with numpy — it is input generation, not the solver — and
draws the same default_rng stream in the same order as the reference
(G(m x n) -> U1, G(n x n) -> V, w(n) -> x, z(m) -> r), so on the same
BLAS it produces the same bytes as the reference's instances.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp


@dataclass
class Truth:
    """problems.py:19-24."""

    x: np.ndarray
    r: np.ndarray
    kappa: float
    beta: float  # ||r(x)||


@dataclass
class LsProblem:
    """problems.py:27-35."""

    a: np.ndarray
    b: np.ndarray
    truth: Truth | None = None

    @property
    def shape(self) -> tuple[int, int]:
        return self.a.shape


def _stiefel_signed(g: np.ndarray) -> np.ndarray:
    """Orthonormal factor of a Gaussian block with the R-diagonal sign
    correction that makes it Haar distributed (problems.py:45-62)."""
    q, r = np.linalg.qr(g, mode="reduced")
    s = np.sign(np.diag(r))
    s[s == 0] = 1.0
    return q * s


def gen_randsvd(m: int, n: int, kappa: float, beta: float, seed: int) -> LsProblem:
    """A = U1 diag(sigma) V' with sigma_j = kappa^(-j/(n-1)), unit-norm planted
    x, residual of norm beta orthogonal to range(A) (problems.py:65-89)."""
    if not (m > n >= 2):
        raise ValueError(f"need m > n >= 2, got m={m}, n={n}")
    if kappa < 1:
        raise ValueError(f"need kappa >= 1, got {kappa}")
    if beta < 0:
        raise ValueError(f"need beta >= 0, got {beta}")
    rng = np.random.default_rng(seed)
    u1 = _stiefel_signed(rng.standard_normal((m, n)))
    v = _stiefel_signed(rng.standard_normal((n, n)))
    sigma = kappa ** (-np.arange(n) / (n - 1))
    a = (u1 * sigma) @ v.T
    w = rng.standard_normal(n)
    x = w / np.linalg.norm(w)
    z = rng.standard_normal(m)
    p = z - u1 @ (u1.T @ z)
    p -= u1 @ (u1.T @ p)
    r = beta * p / np.linalg.norm(p)
    b = a @ x + r
    return LsProblem(a=a, b=b, truth=Truth(x=x, r=r, kappa=float(kappa), beta=float(beta)))


def gen_sparse(m: int, n: int, seed: int) -> LsProblem:
    """Sparse +-1 instance (problems.py:92-110; section 3.5): three
    distinct uniform column positions per row — rows with a repeated position
    are redrawn whole, in stream order, until none is left — values +-1,
    Gaussian b, no ground truth.  CSR with sorted column indices."""
    if not (m >= n >= 3):
        raise ValueError(f"need m >= n >= 3, got m={m}, n={n}")
    rng = np.random.default_rng(seed)
    cols = rng.integers(0, n, size=(m, 3))
    while True:
        s = np.sort(cols, axis=1)
        dup = (s[:, 1:] == s[:, :-1]).any(axis=1)
        if not dup.any():
            break
        cols[dup] = rng.integers(0, n, size=(int(dup.sum()), 3))
    vals = rng.choice(np.array([-1.0, 1.0]), size=(m, 3))
    a = sp.csr_matrix((vals.ravel(), cols.ravel(), 3 * np.arange(m + 1)), shape=(m, n))
    a.sort_indices()
    return LsProblem(a=a, b=rng.standard_normal(m), truth=None)

"""GPU-scale problem instances: `gen_randsvd` on the device plus an on-disk
instance format (SURVEY.md §8(f)-2, §8(d) "C4 instance").

The host generator (problems.gen_randsvd, a restatement of
/root/reference/pkg/src/itsketch/problems.py:65-89) needs ~3 copies of A in
host RAM and hours of single-node LAPACK at C4 (4e6 x 2000, 64 GB).  This
module builds the same construction on the GPU:

    U1 = sign-fixed orthonormal factor of an m x n Gaussian  (problems.py:55-62)
    V  = Haar n x n orthogonal                               (problems.py:45-52)
    sigma_j = kappa^(-j/(n-1)),  A = U1 diag(sigma) V'       (problems.py:80-81)
    x  = w/||w||,  r = beta p/||p||, p = z projected twice onto range(U1)^perp
    b  = A x + r                                             (problems.py:82-88)

U1 comes from CholeskyQR2 of the Gaussian (two Gram / Cholesky / triangular
solve sweeps, row-blocked, in place inside A's buffer).  A tall Gaussian is
well conditioned (kappa(G) ~ 1 + 2 sqrt(n/m)), so the second sweep leaves
||U1'U1 - I|| at the u level, and the Cholesky factor has a positive diagonal,
which is exactly the reference's sign correction (the QR with diag(R) > 0 is
unique).  The draws are Philox streams of torch, not numpy's PCG64, so the
bytes differ from the host generator's: this is test data with the same
distribution, used where the host generator is infeasible.  Every rank of a
row-sharded run can build the same instance (generation blocks are seeded by
(seed, stream, block index), so the result does not depend on the memory
blocking) or load its rows of a saved one.

This is input generation, not the solver: it uses torch's library kernels
(cuRAND Philox, cuBLAS DGEMM, cuSOLVER) and runs on CPU tensors as well.
"""

from __future__ import annotations

import json
import os

import numpy as np
import torch

from .problems import LsProblem, Truth

GEN_BLOCK = 1 << 16          # rows per seeded generation block
_WORK_BYTES = 1 << 30        # row-block temporaries (~1 GB)

_S_GAUSS, _S_HAAR, _S_X, _S_Z = 0, 1, 2, 3


def _seed_of(seed: int, stream: int, block: int) -> int:
    """SplitMix64 of (seed, stream, block) -> Philox seed."""
    v = (int(seed) * 0x9E3779B97F4A7C15 + stream * 0xBF58476D1CE4E5B9 + block * 0x94D049BB133111EB
         + 0x2545F4914F6CDD1D) & 0xFFFFFFFFFFFFFFFF
    v ^= v >> 30
    v = (v * 0xBF58476D1CE4E5B9) & 0xFFFFFFFFFFFFFFFF
    v ^= v >> 27
    v = (v * 0x94D049BB133111EB) & 0xFFFFFFFFFFFFFFFF
    v ^= v >> 31
    return v & 0x7FFFFFFFFFFFFFFF


def _gaussian_rows(out: torch.Tensor, row0: int, seed: int, stream: int) -> None:
    """Fill out = G[row0 : row0 + out.shape[0]] of the (seed, stream) Gaussian,
    block by block; row0 must be a multiple of GEN_BLOCK."""
    if row0 % GEN_BLOCK:
        raise ValueError("row0 must be a multiple of GEN_BLOCK")
    g = torch.Generator(device=out.device)
    rows = out.shape[0]
    for off in range(0, rows, GEN_BLOCK):
        g.manual_seed(_seed_of(seed, stream, (row0 + off) // GEN_BLOCK))
        out[off:off + GEN_BLOCK].normal_(generator=g)


def _blk(n: int) -> int:
    return max(GEN_BLOCK, (_WORK_BYTES // (8 * max(n, 1))) // GEN_BLOCK * GEN_BLOCK)


def _gram(u: torch.Tensor) -> torch.Tensor:
    m, n = u.shape
    g = torch.zeros((n, n), dtype=u.dtype, device=u.device)
    for i in range(0, m, _blk(n)):
        ub = u[i:i + _blk(n)]
        g.addmm_(ub.T, ub)
    return g


def _right_solve_inplace(u: torch.Tensor, r: torch.Tensor) -> None:
    """u <- u R^-1 (R upper triangular), row block by row block."""
    for i in range(0, u.shape[0], _blk(u.shape[1])):
        ub = u[i:i + _blk(u.shape[1])]
        ub.copy_(torch.linalg.solve_triangular(r, ub, upper=True, left=False))


def cholesky_qr2_inplace(u: torch.Tensor) -> torch.Tensor:
    """Orthonormalise the columns of the tall matrix `u` in place (CholeskyQR2);
    returns the combined triangular factor R (diag > 0) with G = U R."""
    r1 = torch.linalg.cholesky(_gram(u), upper=True)
    _right_solve_inplace(u, r1)
    r2 = torch.linalg.cholesky(_gram(u), upper=True)
    _right_solve_inplace(u, r2)
    return r2 @ r1


def _project_out(u: torch.Tensor, z: torch.Tensor) -> torch.Tensor:
    """z - U (U' z), row-blocked."""
    n = u.shape[1]
    c = torch.zeros(n, dtype=u.dtype, device=u.device)
    for i in range(0, u.shape[0], _blk(n)):
        c.addmv_(u[i:i + _blk(n)].T, z[i:i + _blk(n)])
    p = z.clone()
    for i in range(0, u.shape[0], _blk(n)):
        p[i:i + _blk(n)].sub_(u[i:i + _blk(n)] @ c)
    return p


def gen_randsvd_device(m: int, n: int, kappa: float, beta: float, seed: int,
                       device: torch.device | str | None = None) -> LsProblem:
    """The gen_randsvd construction (problems.py:65-89) on `device`.

    Returns an LsProblem whose `a`, `b` and `truth.r` are fp64 tensors on the
    device (A row-major, contiguous) and `truth.x` a host numpy vector.  Peak
    device memory is A plus ~1 GB of row-block temporaries."""
    if not (m > n >= 2):
        raise ValueError(f"need m > n >= 2, got m={m}, n={n}")
    if kappa < 1:
        raise ValueError(f"need kappa >= 1, got {kappa}")
    if beta < 0:
        raise ValueError(f"need beta >= 0, got {beta}")
    dev = torch.device(device) if device is not None else (
        torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else torch.device("cpu"))
    f64 = dict(dtype=torch.float64, device=dev)
    a = torch.empty((m, n), **f64)
    _gaussian_rows(a, 0, seed, _S_GAUSS)
    cholesky_qr2_inplace(a)                                   # a holds U1
    gv = torch.empty((n, n), **f64)
    _gaussian_rows(gv, 0, seed, _S_HAAR)
    q, rv = torch.linalg.qr(gv)
    s = torch.sign(torch.diagonal(rv))
    s[s == 0] = 1.0
    v = q * s
    sigma = torch.tensor(kappa ** (-np.arange(n) / (n - 1)), **f64)
    w = torch.empty(n, **f64)
    _gaussian_rows(w.view(n, 1), 0, seed, _S_X)
    x = w / torch.linalg.vector_norm(w)
    z = torch.empty(m, **f64)
    _gaussian_rows(z.view(m, 1), 0, seed, _S_Z)
    p = _project_out(a, z)
    p = _project_out(a, p)
    r = beta * p / torch.linalg.vector_norm(p)
    del z, p
    sv = sigma[:, None] * v.T                                  # diag(sigma) V'
    b = torch.empty(m, **f64)
    for i in range(0, m, _blk(n)):
        ab = a[i:i + _blk(n)]
        ab.copy_(ab @ sv)                                      # rows of U1 -> rows of A
        torch.addmv(r[i:i + _blk(n)], ab, x, out=b[i:i + _blk(n)])
    truth = Truth(x=x.cpu().numpy(), r=r, kappa=float(kappa), beta=float(beta))
    return LsProblem(a=a, b=b, truth=truth)


# --------------------------------------------------------------------------
# on-disk instance format: one directory, raw .npy arrays + manifest.json
# --------------------------------------------------------------------------

MANIFEST = "manifest.json"
FORMAT = "itsk-instance-v1"


def _to_host(t) -> np.ndarray:
    return t.detach().cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)


def save_instance(path: str, prob: LsProblem, **meta) -> str:
    """Write A.npy, b.npy, x.npy, r.npy (fp64, C order) and manifest.json.
    A is streamed to disk in row blocks so a device-resident A never needs a
    full host copy."""
    os.makedirs(path, exist_ok=True)
    m, n = (int(s) for s in prob.a.shape)
    mm = np.lib.format.open_memmap(os.path.join(path, "A.npy"), mode="w+", dtype=np.float64, shape=(m, n))
    blk = _blk(n)
    for i in range(0, m, blk):
        mm[i:i + blk] = _to_host(prob.a[i:i + blk])
    mm.flush()
    del mm
    np.save(os.path.join(path, "b.npy"), _to_host(prob.b).astype(np.float64, copy=False))
    man = {"format": FORMAT, "m": m, "n": n, "dtype": "float64", "order": "C",
           "files": {"a": "A.npy", "b": "b.npy"}}
    if prob.truth is not None:
        np.save(os.path.join(path, "x.npy"), _to_host(prob.truth.x))
        np.save(os.path.join(path, "r.npy"), _to_host(prob.truth.r))
        man["files"].update(x="x.npy", r="r.npy")
        man["kappa"], man["beta"] = prob.truth.kappa, prob.truth.beta
    man.update(meta)
    with open(os.path.join(path, MANIFEST), "w") as f:
        json.dump(man, f, indent=1, sort_keys=True)
    return path


def load_instance(path: str, rows: tuple[int, int] | None = None, mmap: bool = True) -> LsProblem:
    """Read an instance (or the row block `rows` = (r0, r1) of it, the shard a
    rank owns; truth.r is sliced the same way, truth.x is whole)."""
    with open(os.path.join(path, MANIFEST)) as f:
        man = json.load(f)
    if man.get("format") != FORMAT:
        raise ValueError(f"{path}: not an {FORMAT} directory")
    mode = "r" if mmap else None
    files = man["files"]
    a = np.load(os.path.join(path, files["a"]), mmap_mode=mode)
    b = np.load(os.path.join(path, files["b"]), mmap_mode=mode)
    if a.shape != (man["m"], man["n"]) or b.shape != (man["m"],):
        raise ValueError(f"{path}: array shapes do not match the manifest")
    sl = slice(None) if rows is None else slice(int(rows[0]), int(rows[1]))
    truth = None
    if "x" in files:
        x = np.load(os.path.join(path, files["x"]))
        r = np.load(os.path.join(path, files["r"]), mmap_mode=mode)
        truth = Truth(x=x, r=r[sl], kappa=float(man["kappa"]), beta=float(man["beta"]))
    return LsProblem(a=a[sl], b=b[sl], truth=truth)

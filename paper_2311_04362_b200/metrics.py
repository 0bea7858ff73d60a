"""Error metrics recorded in the solve trace (itsketch.metrics, metrics.py:31-129).

FE and RE are fused into the solver's device kernels (loop.cu k_control and
the fused pass).  The optimal backward error (Waldén–Karlsson–Sun, metrics.py:
99-129) is an opt-in diagnostic (cfg.track_be, m <= 4000 as in the reference);
it runs on the device through torch.linalg (cuSOLVER) — a library call, off the
hot path.
"""

from __future__ import annotations

import numpy as np
import torch


def forward_error(x_true, x_hat) -> float:
    """||x - x_hat|| / ||x|| (metrics.py:31-37)."""
    x_true = np.asarray(x_true, dtype=float)
    nx = np.linalg.norm(x_true)
    if nx == 0.0:
        raise ValueError("forward_error: true solution has zero norm")
    return float(np.linalg.norm(x_true - np.asarray(x_hat, dtype=float)) / nx)


def residual_error(r_true, r_hat) -> float:
    """||r - r_hat|| / ||r|| (metrics.py:40-46)."""
    r_true = np.asarray(r_true, dtype=float)
    nr = np.linalg.norm(r_true)
    if nr == 0.0:
        raise ValueError("residual_error: true residual has zero norm (consistent system)")
    return float(np.linalg.norm(r_true - np.asarray(r_hat, dtype=float)) / nr)


def backward_error_device(a: torch.Tensor, b: torch.Tensor, x: torch.Tensor, max_m: int = 4000) -> float:
    """metrics.py:99-129 on device tensors."""
    m, n = a.shape
    if m > max_m:
        raise ValueError(f"backward_error capped at m <= {max_m}, got m = {m}")
    nx = torch.linalg.vector_norm(x)
    if float(nx) == 0.0:
        raise ValueError("backward_error requires x_hat != 0")
    r_hat = b - a @ x
    nr = torch.linalg.vector_norm(r_hat)
    if float(nr) == 0.0:
        return 0.0
    nu = nr / nx
    q = r_hat / nr
    if m <= 400:
        eye = torch.eye(m, dtype=a.dtype, device=a.device)
        aug = torch.cat([a, nu * (eye - torch.outer(q, q))], dim=1)
        smin = torch.linalg.svdvals(aug)[-1]
    else:
        qa, ra = torch.linalg.qr(a, mode="reduced")
        pp = qa.T @ q
        tau = torch.linalg.vector_norm(q - qa @ pp)
        z = torch.cat([pp, tau.reshape(1)])
        nz = torch.linalg.vector_norm(z)
        if float(nz) > 0:
            z = z / nz
        eye = torch.eye(n + 1, dtype=a.dtype, device=a.device)
        top = torch.cat([ra.T, torch.zeros((n, 1), dtype=a.dtype, device=a.device)], dim=1)
        f = torch.cat([top, nu * (eye - torch.outer(z, z))], dim=0)
        smin = torch.minimum(nu, torch.linalg.svdvals(f)[-1])
    return float(torch.minimum(nu, smin) / torch.linalg.matrix_norm(a, "fro"))

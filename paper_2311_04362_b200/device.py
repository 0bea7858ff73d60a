"""Device plumbing: tensors in, raw pointers out.

PyTorch provides device memory and streams; every computation on the path is
one of this package's own sm_100a kernels (libitsk_b200.so).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib


def current_device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2311_04362_b200 needs a CUDA (sm_100) device; there is no CPU path")
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr(stream: torch.cuda.Stream | None = None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else int(t.data_ptr())


def as_device_matrix(a, dev: torch.device, non_blocking: bool = True) -> tuple[torch.Tensor, int]:
    """Row-major fp64 matrix on `dev` and its leading dimension (elements).
    numpy / CPU inputs are copied (asynchronously when the host memory is
    pinned); CUDA fp64 tensors with unit column stride are used in place."""
    if isinstance(a, torch.Tensor):
        t = a
        if t.dtype != torch.float64:
            t = t.to(torch.float64)
        if t.device != dev:
            t = t.to(dev, non_blocking=non_blocking)
    else:
        arr = np.asarray(a, dtype=np.float64)
        if arr.ndim != 2:
            raise ValueError(f"expected a matrix, got ndim={arr.ndim}")
        t = torch.from_numpy(np.ascontiguousarray(arr)).to(dev, non_blocking=non_blocking)
    if t.ndim != 2:
        raise ValueError(f"expected a matrix, got ndim={t.ndim}")
    if t.stride(1) != 1 or t.stride(0) < t.shape[1]:
        t = t.contiguous()
    return t, int(t.stride(0)) if t.shape[0] > 1 else int(t.shape[1])


def as_device_vector(v, dev: torch.device, non_blocking: bool = True) -> torch.Tensor:
    if isinstance(v, torch.Tensor):
        t = v.to(device=dev, dtype=torch.float64, non_blocking=non_blocking)
    else:
        arr = np.asarray(v, dtype=np.float64)
        t = torch.from_numpy(np.ascontiguousarray(arr)).to(dev, non_blocking=non_blocking)
    if t.ndim != 1:
        raise ValueError("expected a vector")
    return t.contiguous()


def workspace(nbytes: int, dev: torch.device) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=dev)


def lib(dev: torch.device):
    return _lib.lib_for_device(dev.index if dev.index is not None else torch.cuda.current_device())


def to_numpy(t: torch.Tensor) -> np.ndarray:
    return t.detach().to("cpu").numpy()

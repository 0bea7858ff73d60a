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


# Pageable host memory -> device.  cudaMemcpy from pageable memory is staged by
# the driver on one thread (11.5 GB/s measured on the GPU box); here the rows
# go through two pinned 64 MB buffers filled by torch's multi-threaded host copy
# (61 GB/s on 16 cores) while the previous buffer's copy to the device is in
# flight: 46 GB/s end to end (scripts/h2d_pageable_probe.py).
STAGE_BYTES = 64 << 20
STAGE_MIN_BYTES = 32 << 20   # smaller pageable inputs take the plain copy
_STAGE: dict = {"bufs": None, "evs": [None, None], "next": 0}


def upload_rows_staged(dst: torch.Tensor, src: torch.Tensor, r0: int, r1: int,
                       stream: torch.cuda.Stream) -> torch.cuda.Event | None:
    """dst[r0:r1] (device, row-major fp64) <- src[r0:r1] (pageable CPU fp64
    matrix) through the pinned staging buffers, the device copies on
    `stream`; returns the event of the last one."""
    if _STAGE["bufs"] is None:
        _STAGE["bufs"] = [torch.empty(STAGE_BYTES // 8, dtype=torch.float64, pin_memory=True) for _ in range(2)]
    bufs, evs = _STAGE["bufs"], _STAGE["evs"]
    n = int(src.shape[1])
    rows = max(1, (STAGE_BYTES // 8) // max(n, 1))
    ev = None
    for s0 in range(r0, r1, rows):
        s1 = min(r1, s0 + rows)
        i = _STAGE["next"] & 1
        _STAGE["next"] += 1
        if evs[i] is not None:
            evs[i].synchronize()  # the buffer's previous copy to the device
        hb = bufs[i][: (s1 - s0) * n].view(s1 - s0, n)
        hb.copy_(src[s0:s1])
        with torch.cuda.stream(stream):
            dst[s0:s1].copy_(hb, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(stream)
        evs[i] = ev
    return ev


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
        h = torch.from_numpy(np.ascontiguousarray(arr))
        try:
            t = torch.empty(tuple(h.shape), dtype=torch.float64, device=dev)
        except torch.OutOfMemoryError:
            # a cached block of almost the right size (a previous upload of the
            # same matrix) can neither be reused nor leaves room for a new one
            torch.cuda.empty_cache()
            t = torch.empty(tuple(h.shape), dtype=torch.float64, device=dev)
        if h.numel() * 8 >= STAGE_MIN_BYTES and not h.is_pinned():
            upload_rows_staged(t, h, 0, int(h.shape[0]), torch.cuda.current_stream(dev))
        else:
            t.copy_(h, non_blocking=non_blocking)
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

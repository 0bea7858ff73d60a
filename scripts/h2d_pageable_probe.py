"""Pageable numpy -> device: the driver's own staging (one cudaMemcpy from pageable memory) against staging through
two pinned buffers filled by host threads (numpy releases the GIL in copyto).  python scripts/h2d_pageable_probe.py [GB]"""
import sys, time
from concurrent.futures import ThreadPoolExecutor
import numpy as np, torch
gb = float(sys.argv[1]) if len(sys.argv) > 1 else 4.0
n = 500
m = int(gb * 1e9 / 8 / n)
a = np.random.default_rng(0).standard_normal((m, n))
src = torch.from_numpy(a)
dev = torch.device("cuda")
dst = torch.empty((m, n), dtype=torch.float64, device=dev)
def t(fn, reps=3):
    out = []
    for _ in range(reps):
        torch.cuda.synchronize(); t0 = time.perf_counter(); fn(); torch.cuda.synchronize(); out.append(time.perf_counter() - t0)
    return min(out)
print(f"driver-staged pageable copy: {a.nbytes / t(lambda: dst.copy_(src, non_blocking=True)) / 1e9:.1f} GB/s")
for chunk_mb, nthreads in [(32, 4), (64, 4), (64, 8), (64, 16), (128, 8), (16, 8)]:
    rows = max(1, (chunk_mb << 20) // (8 * n))
    bufs = [torch.empty((rows, n), dtype=torch.float64, pin_memory=True) for _ in range(2)]
    nbufs = [b.numpy() for b in bufs]
    pool = ThreadPoolExecutor(nthreads)
    copy_stream = torch.cuda.Stream()
    def staged():
        evs = [None, None]
        for k, r0 in enumerate(range(0, m, rows)):
            r1 = min(m, r0 + rows); i = k & 1
            if evs[i] is not None: evs[i].synchronize()
            step = -(-(r1 - r0) // nthreads)
            futs = [pool.submit(np.copyto, nbufs[i][s:min(r1 - r0, s + step)], a[r0 + s:min(r1, r0 + s + step)])
                    for s in range(0, r1 - r0, step)]
            for f in futs: f.result()
            with torch.cuda.stream(copy_stream):
                dst[r0:r1].copy_(bufs[i][:r1 - r0], non_blocking=True)
                evs[i] = torch.cuda.Event(); evs[i].record(copy_stream)
    print(f"staged {chunk_mb} MB x2 buffers, {nthreads} threads: {a.nbytes / t(staged) / 1e9:.1f} GB/s", flush=True)
    pool.shutdown()
pin = torch.empty((m, n), dtype=torch.float64, pin_memory=True)
print(f"host copy pageable -> pinned (torch copy_, {torch.get_num_threads()} threads): {a.nbytes / t(lambda: pin.copy_(src)) / 1e9:.1f} GB/s")
print(f"pinned H2D: {a.nbytes / t(lambda: dst.copy_(pin, non_blocking=True)) / 1e9:.1f} GB/s")

"""cuBLAS DGEMM throughput (torch.matmul fp64), the library reference point
for the QR's DMMA tiles: square N^3 and the QR's update shapes at C4
(24000 x k) x (k x 2000).  Best of 10, CUDA events."""
import torch


def bench(m, k, n, reps=10):
    a = torch.randn(m, k, dtype=torch.float64, device="cuda")
    b = torch.randn(k, n, dtype=torch.float64, device="cuda")
    for _ in range(2):
        a @ b
    best = 1e9
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        a @ b
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best, 2.0 * m * k * n / best / 1e9


for shape in [(8192, 8192, 8192), (4096, 4096, 4096), (2000, 24000, 2000), (24000, 64, 2000),
              (24000, 128, 2000), (128, 24000, 2000), (64, 24000, 2000)]:
    ms, tf = bench(*shape)
    print(f"dgemm {shape[0]}x{shape[1]} @ {shape[1]}x{shape[2]}: {ms:.3f} ms  {tf:.2f} TFLOP/s")

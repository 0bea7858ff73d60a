"""Fused-pass timing and agreement over shapes (CUDA events, 30 launches):
    python scripts/pass_ab.py [m,n ...]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2311_04362_b200 import _lib
from bench import fused_pass_timing
shapes = [tuple(int(v) for v in a.split(",")) for a in sys.argv[1:]] or [(4000000, 2000), (1000000, 2000), (2000000, 1000), (500000, 1536)]
lib = _lib.lib_for_device(0)
for m, n in shapes:
    g = torch.Generator(device="cuda").manual_seed(1)
    A = torch.randn(m, n, dtype=torch.float64, device="cuda", generator=g)
    b = torch.randn(m, dtype=torch.float64, device="cuda", generator=g)
    x = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
    ms = fused_pass_timing(lib, A, b, x, 30)
    print(f"pass m={m} n={n}: {ms * 1e3:9.1f} us  "
          f"{8 * m * n / ms / 1e6:7.0f} GB/s", flush=True)
    del A
    torch.cuda.empty_cache()

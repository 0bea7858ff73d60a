import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2311_04362_b200 import _lib
from bench import fused_pass_timing
m, n = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 30
lib = _lib.lib_for_device(0)
A = torch.randn(m, n, dtype=torch.float64, device="cuda")
b = torch.randn(m, dtype=torch.float64, device="cuda")
x = torch.randn(n, dtype=torch.float64, device="cuda")
ms = fused_pass_timing(lib, A, b, x, reps)
print(f"pass m={m} n={n}: {ms*1e3:.1f} us  {8*m*n/ms/1e6:.0f} GB/s")

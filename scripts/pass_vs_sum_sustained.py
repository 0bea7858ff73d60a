"""Sustained streaming under the power cap: the fused pass against torch's A.sum() (a lean read-only reduction)
over the same 64 GB, alternating ~8 s blocks in one process; ms per sweep of A, SM clock and board power.
    python scripts/pass_vs_sum_sustained.py [m n seconds rounds]"""
import os, sys, time, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2311_04362_b200 import _lib
from bench import fused_pass_timing
m, n = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (4000000, 2000)
secs = float(sys.argv[3]) if len(sys.argv) > 3 else 8.0
rounds = int(sys.argv[4]) if len(sys.argv) > 4 else 2
lib = _lib.lib_for_device(0)
g = torch.Generator(device="cuda").manual_seed(1)
A = torch.randn(m, n, dtype=torch.float64, device="cuda", generator=g)
b = torch.randn(m, dtype=torch.float64, device="cuda", generator=g)
x = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
def clock():
    return subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.mem,power.draw", "--format=csv,noheader,nounits"],
                          capture_output=True, text=True).stdout.strip()
def sum_timing(reps):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(reps): A.sum()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
for r in range(rounds):
    for name in ("pass", "sum"):
        t0 = time.time(); ts = []; clk = []
        while time.time() - t0 < secs:
            ts.append(fused_pass_timing(lib, A, b, x, 30) if name == "pass" else sum_timing(30))
            clk.append(clock())
        ms = sum(ts) / len(ts)
        print(f"round {r} {name:4s}: {ms:7.3f} ms per sweep ({8e-6 * m * n / ms:6.0f} GB/s); sm MHz, mem MHz, W: {clk[len(clk) // 2]} | {clk[-1]}", flush=True)

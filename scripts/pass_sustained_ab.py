"""Sustained A/B of two pass kernels in one process (the power cap decides):
alternate ~8 s blocks of back-to-back C4 passes, report ms per pass and the SM clock.
    python scripts/pass_sustained_ab.py ENVNAME [m n seconds rounds]
(needs a build with an environment switch between the two kernels; the product library has none)"""
import ctypes, os, sys, time, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2311_04362_b200 import _lib
from bench import fused_pass_timing
env = sys.argv[1]
m, n = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (4000000, 2000)
secs = float(sys.argv[4]) if len(sys.argv) > 4 else 8.0
rounds = int(sys.argv[5]) if len(sys.argv) > 5 else 3
lib = _lib.lib_for_device(0)
g = torch.Generator(device="cuda").manual_seed(1)
A = torch.randn(m, n, dtype=torch.float64, device="cuda", generator=g)
b = torch.randn(m, dtype=torch.float64, device="cuda", generator=g)
x = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
def clock():
    out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits"],
                         capture_output=True, text=True).stdout.strip()
    return out
for r in range(rounds):
    for val in ("0", "1"):
        os.environ[env] = val
        t0 = time.time(); ts = []; clk = []
        while time.time() - t0 < secs:
            ts.append(fused_pass_timing(lib, A, b, x, 30))
            clk.append(clock())
        print(f"round {r} {env}={val}: {1e3 * sum(ts) / len(ts):8.1f} us per pass over {30 * len(ts)} launches; last clocks/power {clk[-1]}", flush=True)

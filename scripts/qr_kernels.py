"""Per-kernel device time of the QR alone (torch.profiler / CUPTI, warm):
    python scripts/qr_kernels.py d n [reps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile
from paper_2311_04362_b200 import _lib
from paper_2311_04362_b200 import device as dv
from paper_2311_04362_b200.linalg import qr_workspace

d, n = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
lib = _lib.lib_for_device(0)
ldw = (n + 2) // 2 * 2  # the solver's even leading dimension
W0 = torch.randn(d, ldw, dtype=torch.float64, device="cuda")
W = W0.clone()
R = torch.empty(n, n, dtype=torch.float64, device="cuda")
z = torch.empty(n, dtype=torch.float64, device="cuda")
ws = qr_workspace(d, n, W.device)
s = dv.stream_ptr()


def run():
    W.copy_(W0)
    _lib.check(lib.itsk_qr_aug(dv.ptr(W), d, n, ldw, dv.ptr(R), dv.ptr(z), dv.ptr(ws), ws.numel(), s))


for _ in range(2):
    run()
torch.cuda.synchronize()
ts = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); run(); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print(f"QR d={d} n={n} ldw={ldw}: wall (CUDA events, incl. the W copy) " + " ".join(f"{t:.2f}" for t in ts) + " ms")
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(reps):
        run()
    torch.cuda.synchronize()
agg = {}
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA and e.device_time_total > 0:
        k = e.name.replace("(anonymous namespace)::", "").replace("itsk::", "").split("(")[0][:50]
        c, t = agg.get(k, (0, 0.0))
        agg[k] = (c + 1, t + e.device_time_total)
print(f"QR d={d} n={n}: per QR, warm, {reps} reps (kernels on 3 streams overlap: the sum exceeds the wall time)")
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:50s} {c / reps:7.1f} launches {t / reps:10.1f} us  {t / c:8.2f} us each")

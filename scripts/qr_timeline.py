"""Per-stream kernel timeline of one warm QR (torch.profiler / CUPTI chrome
trace): busy time and gaps per stream, and where the critical (panel)
stream waits.  python scripts/qr_timeline.py d n"""
import json, os, sys, tempfile
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile
from paper_2311_04362_b200 import _lib
from paper_2311_04362_b200 import device as dv
from paper_2311_04362_b200.linalg import qr_workspace

d, n = int(sys.argv[1]), int(sys.argv[2])
lib = _lib.lib_for_device(0)
ldw = (n + 2) // 2 * 2
W0 = torch.randn(d, ldw, dtype=torch.float64, device="cuda")
W = W0.clone()
R = torch.empty(n, n, dtype=torch.float64, device="cuda")
z = torch.empty(n, dtype=torch.float64, device="cuda")
ws = qr_workspace(d, n, W.device)
s = dv.stream_ptr()


def run():
    W.copy_(W0)
    _lib.check(lib.itsk_qr_aug(dv.ptr(W), d, n, ldw, dv.ptr(R), dv.ptr(z), dv.ptr(ws), ws.numel(), s))


for _ in range(3):
    run()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    run()
    torch.cuda.synchronize()
path = os.path.join(tempfile.gettempdir(), "qr_trace.json")
prof.export_chrome_trace(path)
ev = [e for e in json.load(open(path))["traceEvents"] if e.get("cat") == "kernel"]
ev.sort(key=lambda e: e["ts"])
t0 = ev[0]["ts"]
t1 = max(e["ts"] + e["dur"] for e in ev)
print(f"QR d={d} n={n}: {len(ev)} kernels, wall {t1 - t0:.0f} us")
by = {}
for e in ev:
    by.setdefault(e["args"].get("stream"), []).append(e)
for st, es in by.items():
    busy = sum(e["dur"] for e in es)
    names = {}
    for e in es:
        k = e["name"].replace("(anonymous namespace)::", "").replace("itsk::", "").split("(")[0][:28]
        names[k] = names.get(k, 0.0) + e["dur"]
    top = ", ".join(f"{k} {v:.0f}" for k, v in sorted(names.items(), key=lambda x: -x[1])[:5])
    print(f"stream {st}: {len(es)} kernels, busy {busy:.0f} us ({100 * busy / (t1 - t0):.0f} %): {top}")
def short(e):
    return e["name"].replace("(anonymous namespace)::", "").replace("itsk::", "").replace("void ", "").split("(")[0][:22]


# the panel stream: gaps between consecutive kernels, largest first, and what preceded them
pst = next(st for st, es in by.items() if any("k_qr_panel" in e["name"] for e in es))
es = by[pst]
gaps = []
for a, b in zip(es, es[1:]):
    g = b["ts"] - (a["ts"] + a["dur"])
    gaps.append((g, short(a), short(b), a["ts"] - t0))
tot = sum(g for g, *_ in gaps)
print(f"panel stream {pst}: gaps total {tot:.0f} us; largest:")
for g, a, b, t in sorted(gaps, reverse=True)[:12]:
    print(f"  {g:8.1f} us at {t:8.0f}: after {a} before {b}")
hist = {}
for g, a, b, t in gaps:
    key = (a, b)
    c, sm = hist.get(key, (0, 0.0))
    hist[key] = (c + 1, sm + g)
print("gap totals by (before, after):")
for (a, b), (c, sm) in sorted(hist.items(), key=lambda x: -x[1][1])[:8]:
    print(f"  {a:>24s} -> {b:24s} {c:4d} x, {sm:8.0f} us")

# what the chain waited for: for each gap > 20 us, the kernels of other
# streams that ended inside it (the last one released the chain)
print("chain gaps > 20 us and the other streams' kernels ending inside them:")
other = [e for st, es in by.items() if st != pst for e in es]
cat = {}
for a, b in zip(es, es[1:]):
    g0, g1 = a["ts"] + a["dur"], b["ts"]
    if g1 - g0 < 20:
        continue
    inside = sorted((e for e in other if g0 <= e["ts"] + e["dur"] <= g1), key=lambda e: e["ts"] + e["dur"])
    tail = " | ".join(f"{short(e)}@s{e['args'].get('stream')} {e['ts'] + e['dur'] - g0:.0f}" for e in inside[-4:])
    key = short(inside[-1]) if inside else "-"
    c, sm = cat.get(key, (0, 0.0))
    cat[key] = (c + 1, sm + g1 - g0)
    print(f"  {g1 - g0:7.1f} us {short(a)} -> {short(b)}: {tail}")
print("gap totals by the kernel that ended last inside:")
for k, (c, sm) in sorted(cat.items(), key=lambda x: -x[1][1]):
    print(f"  {k:24s} {c:4d} x {sm:8.0f} us")

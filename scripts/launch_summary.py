"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list:
per-kernel count, total and mean duration (cold-cache, serialised: compare
shares, not absolute times)."""
import csv, io, re, sys
path = sys.argv[1]
txt = open(path).read()
start = txt.find('"ID"')
rows = list(csv.DictReader(io.StringIO(txt[start:])))
agg = {}
for r in rows:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(.*", "", r["Kernel Name"]).replace("itsk::<unnamed>::", "").strip()
    v = float(r["Metric Value"].replace(",", ""))
    unit = r.get("Metric Unit", "")
    v = v / 1000.0 if unit in ("nsecond", "ns") else (v if unit in ("usecond", "us") else v * 1000.0 if unit == "msecond" else v)
    c, t = agg.get(name, (0, 0.0))
    agg[name] = (c + 1, t + v)
tot = sum(t for _, t in agg.values())
print(f"{'kernel':60s} {'count':>6s} {'total us':>10s} {'mean us':>9s} {'share':>6s}")
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k[:60]:60s} {c:6d} {t:10.1f} {t / c:9.2f} {100 * t / tot:5.1f}%")
print(f"{'total':60s} {sum(c for c, _ in agg.values()):6d} {tot:10.1f}")

"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list."""
import csv, sys
from collections import defaultdict
rows = list(csv.reader(open(sys.argv[1])))
hdr = None; data = []
for r in rows:
    if r and r[0] == 'ID': hdr = r; continue
    if hdr and len(r) == len(hdr): data.append(dict(zip(hdr, r)))
frac = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
data = data[int(len(data) * frac):]
agg = defaultdict(lambda: [0, 0.0])
for d in data:
    nm = d['Kernel Name'].replace('itsk::<unnamed>::', '').replace('(anonymous namespace)::', '')[:70]
    agg[nm][0] += 1; agg[nm][1] += float(d['Metric Value'])
tot = sum(v[1] for v in agg.values())
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{v[1]/1e3:9.1f} us {v[0]:4d} x {v[1]/1e3/v[0]:8.1f} us  {100*v[1]/tot:5.1f}%  {k}")
print(f"total {tot/1e3:.1f} us over {len(data)} launches")

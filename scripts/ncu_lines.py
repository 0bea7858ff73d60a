"""Map ncu per-instruction stall samples to CUDA source lines via nvdisasm -g.
usage: ncu_lines.py report.ncu-rep object.o kernel_substring source.cu [top]"""
import csv, re, subprocess, sys, os, tempfile
rep, obj, kname, srcf = sys.argv[1:5]
top = int(sys.argv[5]) if len(sys.argv) > 5 else 30
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv'], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[1]; rows = [x for x in r[2:] if len(x) > 3]
i_s = h.index('Warp Stall Sampling (All Samples)')
base = int(rows[0][0], 16)
samples = {int(x[0], 16) - base: int(x[i_s] or 0) for x in rows}
td = tempfile.mkdtemp()
subprocess.run(['cuobjdump', '-xelf', 'all', os.path.abspath(obj)], cwd=td, capture_output=True)
cub = [os.path.join(td, f) for f in os.listdir(td) if f.endswith('.cubin')][0]
txt = subprocess.run(['nvdisasm', '-g', '-c', cub], capture_output=True, text=True).stdout
secs = re.split(r'\n//-+ \.text\.', txt)
sec = [s for s in secs if s.split()[0].find(kname) >= 0][0]
line = None; agg = {}
for ln in sec.splitlines():
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        line = (os.path.basename(m.group(1)), int(m.group(2))); continue
    m2 = re.match(r'\s*/\*([0-9a-f]{4,})\*/', ln)
    if m2 and line is not None:
        agg[line] = agg.get(line, 0) + samples.get(int(m2.group(1), 16), 0)
tot = sum(samples.values())
print('samples', tot, 'mapped', sum(agg.values()))
src = open(srcf).read().splitlines()
for (f, l), v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
    s = src[l - 1].strip()[:95] if f == os.path.basename(srcf) else ''
    print(f"{v:6d} {100*v/tot:5.1f}% {f}:{l:<4d} {s}")

"""Summarise an ncu --csv launch list (gpu__time_duration.sum per kernel)."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = None; out = []
for r in rows:
    if 'Kernel Name' in r: hdr = r; continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get('Metric Name') == 'gpu__time_duration.sum':
            out.append((d['Kernel Name'].split('(')[0].replace('void ', ''), d.get('Grid Size', ''), float(d['Metric Value'])))
tot = sum(o[2] for o in out)
for i, (n, g, v) in enumerate(out):
    print(f"{i:3d} {n:28s} {g:16s} {v/1e3:8.2f} us")
print(f"kernels {len(out)}  sum {tot/1e3:.1f} us")
by = {}
for n, g, v in out: by[n] = by.get(n, 0) + v
for n, v in sorted(by.items(), key=lambda x: -x[1]): print(f"  {n:28s} {v/1e3:8.1f} us  {v/tot*100:5.1f}%")

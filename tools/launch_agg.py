"""Aggregate an ncu --csv launch list (time + DRAM bytes) per kernel/grid over
the Comps that follow the last plan build (k_plain)."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = None; d = {}; order = []
for r in rows:
    if 'Kernel Name' in r: hdr = r; continue
    if hdr and len(r) == len(hdr):
        x = dict(zip(hdr, r)); key = int(x['ID'])
        if key not in d:
            d[key] = {'name': x['Kernel Name'].split('(')[0].replace('void ', ''), 'grid': x['Grid Size']}
            order.append(key)
        d[key][x['Metric Name']] = float(x['Metric Value'].replace(',', ''))
last_plan = max([i for i in order if d[i]['name'].startswith('k_plain')], default=-1)
sel = [d[i] for i in order if i > last_plan]
ncomp = max(1, sum(1 for x in sel if x['name'] == 'hc::k_cl_intt2<3>'))
agg = {}
for x in sel:
    a = agg.setdefault((x['name'], x['grid']), [0, 0, 0, 0])
    a[0] += 1; a[1] += x.get('gpu__time_duration.sum', 0); a[2] += x.get('dram__bytes_read.sum', 0); a[3] += x.get('dram__bytes_write.sum', 0)
tot = sum(a[1] for a in agg.values())
print(f"comps {ncomp}  launches/comp {len(sel)/ncomp:.0f}  serialised kernel time/comp {tot/ncomp/1e6:.3f} ms")
for (n, g), a in sorted(agg.items(), key=lambda x: -x[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{n:28s} {g:14s} x{a[0]/ncomp:5.1f}/comp {a[1]/a[0]/1e3:9.1f} us/launch {a[1]/tot*100:5.1f}%  rd {a[2]/a[0]/1e6:7.1f} MB wr {a[3]/a[0]/1e6:7.1f} MB")

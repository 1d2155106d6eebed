"""DRAM bytes per launch of one kernel from an `ncu --page raw --csv` dump:
dram__bytes_read.sum + dram__bytes_write.sum, beside its algorithmic bytes.

  python tools/ncu_traffic.py raw.csv 'kernel<...>' jobs_per_launch algorithmic_bytes_per_job
"""
import csv
import io
import json
import sys

raw, name, jobs, per_job = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
rows = list(csv.reader(io.StringIO(open(raw).read())))
hdr, units = rows[0], rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
out = {}
for r in rows[2:]:
    d, u = dict(zip(hdr, r)), dict(zip(hdr, units))
    b = 0.0
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        b += float(d[k].replace(",", "")) * scale.get(u[k], 1)
    dur = float(d["gpu__time_duration.sum"].replace(",", "")) * {"nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6,
                                                                 "msecond": 1e-3, "ms": 1e-3}[u["gpu__time_duration.sum"]]
    out[name] = {
        "dram_bytes_per_launch": b,
        "algorithmic_bytes_per_launch": jobs * per_job,
        "jobs_per_launch": jobs,
        "ncu_duration_s": dur,
        "source": "ncu --set full --clock-control none, one launch inside bench.py's timed region",
    }
    break
print(json.dumps(out, indent=1))

"""Key metrics of one or more ncu reports (ncu -i ... --page raw --csv).

  python tools/ncu_summary.py rep1.ncu-rep [rep2 ...]
"""
import csv, io, subprocess, sys

KEYS = [
    ("gpu__time_duration.sum", "duration (us)", 1e-3),
    ("launch__grid_size", "grid", 1), ("launch__block_size", "block", 1),
    ("launch__registers_per_thread", "regs/thread", 1),
    ("launch__cluster_dim_x", "cluster", 1),
    ("dram__bytes_read.sum", "DRAM read (MB)", 1), ("dram__bytes_write.sum", "DRAM write (MB)", 1),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak", 1),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %", 1),
    ("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed", "fmaheavy pipe % (elapsed)", 1),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe % (active)", 1),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %", 1),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %", 1),
    ("sm__cycles_active.avg", "SM active cycles (avg)", 1),
    ("smsp__average_warp_latency_issue_stalled_barrier", "stall barrier", 1),
]

for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        print(rep, "no data"); continue
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        print(f"== {rep}: {d.get('Kernel Name', '?')[:120]}")
        for k, label, scale in KEYS:
            if k in d and d[k] != "":
                v = d[k]
                try:
                    fv = float(v.replace(",", ""))
                    unit = u.get(k, "")
                    if k.startswith("dram__bytes"):
                        fv = fv * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1, "Gbyte": 1e3}.get(unit, 1)
                    elif k == "gpu__time_duration.sum":
                        fv = fv * {"nsecond": 1e-3, "usecond": 1, "msecond": 1e3}.get(unit, 1)
                    print(f"  {label:28s} {fv:12.3f}")
                except ValueError:
                    print(f"  {label:28s} {v}")

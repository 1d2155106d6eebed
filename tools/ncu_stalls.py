"""Warp-stall breakdown, pipe utilisation and memory counters of ncu reports.
  python tools/ncu_stalls.py rep.ncu-rep [...]"""
import csv, io, subprocess, sys
for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    for r in rows[2:]:
        d = dict(zip(h, r))
        print("==", rep, d.get("Kernel Name", "?")[:80])
        st = sorted(((float(v), k) for k, v in d.items() if "issue_stalled" in k and k.endswith("per_issue_active.ratio")), reverse=True)
        print("  stalls/issue:", ", ".join(f"{k.split('issue_stalled_')[1].split('_per_')[0]} {v:.2f}" for v, k in st[:9]))
        for k in ("gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
                  "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
                  "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
                  "sm__warps_active.avg.pct_of_peak_sustained_active", "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
                  "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
                  "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread", "smsp__inst_executed_op_local_ld.sum",
                  "lts__t_bytes.sum", "l1tex__t_bytes.sum"):
            if d.get(k) not in (None, ""):
                print(f"  {k:70s} {d[k]}")

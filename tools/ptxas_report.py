"""Registers / spills per kernel from `nvcc -Xptxas=-v` (reads stdin).

  nvcc ... -Xptxas=-v ... 2>&1 | python tools/ptxas_report.py [--spills]
"""
import re, subprocess, sys

name, rows = None, []
for line in sys.stdin:
    m = re.search(r"Compiling entry function '([^']+)'", line)
    if m:
        name = m.group(1)
        continue
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and name:
        cur = [name, int(m.group(2)), int(m.group(3)), None]
        rows.append(cur)
        continue
    m = re.search(r"Used (\d+) registers", line)
    if m and rows and rows[-1][0] == name:
        rows[-1][3] = int(m.group(1))
dem = subprocess.run(["c++filt"], input="\n".join(r[0] for r in rows), capture_output=True, text=True).stdout.split("\n")
for r, d in zip(rows, dem):
    if "--spills" in sys.argv and r[1] == 0 and r[2] == 0:
        continue
    print(f"{r[3]!s:>4} regs  spill st/ld {r[1]:>4}/{r[2]:<4}  {d}")

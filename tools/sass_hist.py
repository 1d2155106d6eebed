"""SASS opcode histogram of a kernel's hottest loop (cuobjdump -sass of the
shipped .so): the evidence for "k" = IMAD-pipe instructions per butterfly.

    python tools/sass_hist.py [lib.so] [function-substring] [butterflies-per-iteration]

The loop is the span between the target of the function's last backward
branch and that branch.  Mnemonics are grouped by pipe the way the
microarchitecture notes do: IMAD* / IMUL on the fma-heavy (IMAD) pipe,
IADD3 / LOP3 / SHF / ISETP / SEL / PRMT on the ALU pipe.
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_2408_17063_b200", "libhcomp.so")
fn = sys.argv[2] if len(sys.argv) > 2 else "k_bf_peak"
per_iter = float(sys.argv[3]) if len(sys.argv) > 3 else 16.0

sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
funcs = re.split(r"\n\s*Function : ", sass)
body = next(f for f in funcs[1:] if fn in f.split("\n", 1)[0])
name = body.split("\n", 1)[0].strip()
ins = []
for ln in body.split("\n"):
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
# last backward branch
loop = None
for addr, txt in ins:
    m = re.search(r"\bBRA\b.*?(0x[0-9a-f]+)", txt)
    if m and int(m.group(1), 16) < addr:
        loop = (int(m.group(1), 16), addr)
if loop is None:
    sys.exit(f"{name}: no backward branch")
span = [t for a, t in ins if loop[0] <= a <= loop[1]]
ops = collections.Counter()
for t in span:
    t = re.sub(r"^@!?U?P\w+\s+", "", t)
    ops[t.split()[0]] += 1
imad = sum(v for k, v in ops.items() if k.startswith(("IMAD", "IMUL")))
imad_mov = sum(v for k, v in ops.items() if k.startswith("IMAD.MOV"))
alu = sum(v for k, v in ops.items() if k.split(".")[0] in ("IADD3", "LOP3", "SHF", "ISETP", "SEL", "PRMT", "IADD", "VIADD", "LEA", "MOV", "IABS"))
print(f"{name}\nloop 0x{loop[0]:x}-0x{loop[1]:x}: {len(span)} instructions, {per_iter:g} butterflies per iteration")
for k, v in ops.most_common():
    print(f"  {k:28s} {v:5d}  {v / per_iter:6.2f}/bfly")
print(f"IMAD-pipe (IMAD*, IMUL*): {imad} = {imad / per_iter:.2f} per butterfly (of which IMAD.MOV {imad_mov / per_iter:.2f})")
print(f"ALU-pipe: {alu} = {alu / per_iter:.2f} per butterfly; total {len(span) / per_iter:.2f} per butterfly")

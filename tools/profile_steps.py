"""Per-step timing of the Comp schedule (un-graphed, CUDA events per step).
usage: python tools/profile_steps.py [N] [s] [reps]"""
import os, sys, random, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2408_17063_b200 as P
from paper_2408_17063_b200 import _lib

N = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
s = int(sys.argv[2]) if len(sys.argv) > 2 else 16
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
p = 65537 if N < 65537 else (786433 if N < 786433 else 4423681)
he = P.HeParams(8192, p, 3)
params = P.CompressionParams(N, s, he)
be = P.B200BgvBackend(he, seed=0, noise_guard=False)
keys = be.keygen(*P.plan_rotation_amounts(s, 8192))
rng = np.random.default_rng(1)
C = params.num_ciphertexts
cd = np.stack([np.stack([rng.integers(0, q, 8192, dtype=np.uint64) for q in be.q]) for _ in range(2 * C)]).reshape(C, 2, 4, 8192)
cv = cd.copy()
dc = P.DeviceComp(be, params, keys)
dc.set_inputs(cd, cv)
L = _lib.lib(); h = be._ctx()
for _ in range(3):
    dc.launch()
dc.output()
ms = np.zeros(4096, np.float32); kind = np.zeros(4096, np.int32); jobs = np.zeros(4096, np.int32)
names = {0: "xform", 1: "compose", 2: "ksmac", 3: "diagx", 4: "sumcopies", 5: "memset", 6: "intt2"}
for r in range(reps):
    n = L.hc_comp_profile(h, None, 4096, _lib.ptr(ms), _lib.ptr(kind), _lib.ptr(jobs))
print("plan", be.plan_info())
tot = 0
for i in range(n):
    tot += ms[i]
    print(f"{i:3d} {names[int(kind[i])]:9s} jobs={int(jobs[i]):5d} {ms[i]*1e3:8.1f} us")
print("total ms", tot)
import torch
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(50):
    dc.launch()
dc.output()
print("graph ms/comp", (time.perf_counter() - t0) / 50 * 1e3)
agg = {}
for i in range(n):
    k = (names[int(kind[i])], int(jobs[i]))
    c, t = agg.get(k, (0, 0.0))
    agg[k] = (c + 1, t + float(ms[i]))
print("by (kind, jobs): count, total us, us/job")
for (nm, j), (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"  {nm:9s} jobs={j:5d} x{c:4d} {t*1e3:9.1f} us  {t*1e3/max(1,c*j):7.2f} us/job")

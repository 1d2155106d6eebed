"""Per-fold phase timeline of the persistent fold chain k_foldchain (needs
libhcomp_trace.so: nvcc ... -DHC_TRACE -DHC_MAXL=3).  Points: 0 fold start
(after the grid barrier), 1 res_f.c1 loaded, 2 GS passes, 3 INTT all-to-all,
4 half exchange, 5 digits composed, 6 cluster barrier, 7 digits gathered
(DSMEM), 8 NTT all-to-all, 9 NTT passes, 10 key MAC, 11 c0 slack done."""
import os, sys
HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ.setdefault("HCOMP_LIB", os.path.join(HERE, "paper_2408_17063_b200", "libhcomp_trace.so"))
sys.path.insert(0, HERE)
import numpy as np, torch
import paper_2408_17063_b200 as P
from paper_2408_17063_b200 import _lib
N = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
s = int(sys.argv[2]) if len(sys.argv) > 2 else 16
he = P.HeParams(8192, 65537, 3); params = P.CompressionParams(N, s, he)
be = P.B200BgvBackend(he, seed=0, noise_guard=False)
keys = be.keygen(*P.plan_rotation_amounts(s, 8192))
rng = np.random.default_rng(1); C = params.num_ciphertexts
cd = np.stack([np.stack([rng.integers(0, q, 8192, dtype=np.uint64) for q in be.q]) for _ in range(2 * C)]).reshape(C, 2, 4, 8192)
dc = P.DeviceComp(be, params, keys); dc.set_inputs(cd, cd.copy())
L = _lib.lib()
for _ in range(5): dc.launch()
torch.cuda.synchronize()
tr = np.zeros((12, 128, 12), dtype=np.uint64)
_lib.check(L.hc_trace_read_tail(_lib.ptr(tr)))
t0 = tr[0][:, 0][tr[0][:, 0] > 0].min()
names = ["start", "loaded", "GS", "a2a", "half", "digits", "clbar", "gather", "ntt-x", "passes", "mac", "slack"]
for f in range(12):
    b = tr[f].astype(np.int64)
    live = b[:, 0] > 0
    if not live.any():
        break
    b = b[live]
    med = [(np.median(b[:, i]) - t0) / 1e3 for i in range(12)]
    mx = [(b[:, i].max() - t0) / 1e3 for i in range(12)]
    print(f"fold {f}: " + " ".join(f"{n} {m:6.2f}" for n, m in zip(names, med)) + f" | max slack {mx[11]:6.2f}")
if "--clusters" in sys.argv:  # per-cluster medians of the first two folds (cluster d = CTAs 16d .. 16d+15)
    for f in range(2):
        b = tr[f].astype(np.int64)
        for d in range(8):
            rows = b[16 * d:16 * d + 16]
            rows = rows[rows[:, 0] > 0]
            if len(rows):
                print(f"fold {f} cluster {d}: " + " ".join(f"{n} {(np.median(rows[:, i]) - t0) / 1e3:6.2f}" for i, n in enumerate(names)))

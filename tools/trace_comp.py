"""Per-launch phase timeline of one Comp graph run (needs libhcomp_trace.so:
nvcc ... -DHC_TRACE -DHC_MAXL=3 -o paper_2408_17063_b200/libhcomp_trace.so)."""
import os, sys
HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ.setdefault("HCOMP_LIB", os.path.join(HERE, "paper_2408_17063_b200", "libhcomp_trace.so"))
sys.path.insert(0, HERE)
import numpy as np, torch
import paper_2408_17063_b200 as P
from paper_2408_17063_b200 import _lib
N = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
s = int(sys.argv[2]) if len(sys.argv) > 2 else 16
p = 65537 if N < 65537 else 786433
he = P.HeParams(8192, p, 3); params = P.CompressionParams(N, s, he)
be = P.B200BgvBackend(he, seed=0, noise_guard=False)
keys = be.keygen(*P.plan_rotation_amounts(s, 8192))
rng = np.random.default_rng(1); C = params.num_ciphertexts
cd = np.stack([np.stack([rng.integers(0, q, 8192, dtype=np.uint64) for q in be.q]) for _ in range(2 * C)]).reshape(C, 2, 4, 8192)
if os.environ.get("TRACE_LANES"): _lib.lib().hc_set_lane_blocks(int(os.environ["TRACE_LANES"]))
dc = P.DeviceComp(be, params, keys); dc.set_inputs(cd, cd.copy())
L = _lib.lib()
L.hc_trace_reset()
for _ in range(5): dc.launch()
torch.cuda.synchronize()
tr = np.zeros((128, 512, 8), dtype=np.uint64)
_lib.check(L.hc_trace_read(_lib.ptr(tr)))
t0 = None
rows = []
for lid in range(64):
    blk = tr[lid]
    st = blk[:, 0]
    live = st > 0
    if not live.any(): continue
    b = blk[live].astype(np.int64)
    s0 = b[:, 0].min(); e = b[:, 5].max() if (b[:, 5] > 0).any() else b[:, 1].max()
    rows.append((lid, s0, e, b))
t0 = min(r[1] for r in rows)
prev_end = t0
for lid, s0, e, b in rows:
    def med(i, j):
        m = (b[:, i] > 0) & (b[:, j] > 0)
        return np.median(b[m, j] - b[m, i]) / 1e3 if m.any() else float('nan')
    print(f"launch {lid:3d} blocks {len(b):4d} start {(s0-t0)/1e3:8.2f} gap {(s0-prev_end)/1e3:6.2f} dur {(e-s0)/1e3:7.2f} us | "
          f"ld {med(0,1):5.2f} 1->4 {med(1,4):5.2f} 4->5 {med(4,5):5.2f} start-spread {(b[:,0].max()-s0)/1e3:5.2f}"
          + (f" | 0->6 {med(0,6):5.2f} 6->7 {med(6,7):5.2f} 7->1 {med(7,1):5.2f}" if (b[:, 6] > 0).any() else "")
          + (f" | 4->3 {med(4,3):5.2f} 3->5 {med(3,5):5.2f}" if (b[:, 3] > b[:, 4]).all() else ""))
    prev_end = e
print("total", (prev_end - t0) / 1e3, "us")

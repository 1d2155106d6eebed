"""Single-CTA transform throughput: 1024-thread (one per SM) vs the 256-thread
three-per-SM variant (hc_set_vt2_jobs)."""
import os, sys, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_17063_b200 as P
from paper_2408_17063_b200 import _lib
be = P.B200BgvBackend(P.HeParams(8192, 65537, 3), seed=0)
L = _lib.lib(); h = be._ctx()
L.hc_set_cluster_threshold(0)
for vt in (1 << 30, 1):  # one per SM, then two per SM everywhere
    L.hc_set_vt2_jobs(vt)
    for dirn in (0, 1):
        for nj in (148, 296, 592, 1184):
            us = ctypes.c_double()
            _lib.check(L.hc_bench_xform(h, nj, dirn, 30, ctypes.byref(us)))
            print(f"vt2>={vt:10d} dir {dirn} jobs {nj:5d}: {us.value:8.2f} us  {nj*4096*13/(us.value*1e-6)/1e9:6.1f} Gbfly/s", flush=True)
L.hc_set_vt2_jobs(200)
L.hc_set_cluster_threshold(48)

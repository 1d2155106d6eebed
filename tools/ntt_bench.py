"""Transform kernel microbenchmark: latency (1 job) and throughput (many jobs)."""
import os, sys, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_17063_b200 as P
from paper_2408_17063_b200 import _lib
be = P.B200BgvBackend(P.HeParams(8192, 65537, 3), seed=0)
L = _lib.lib(); h = be._ctx()
pk = ctypes.c_double()
_lib.check(L.hc_bf_peak(h, ctypes.byref(pk)))
print(f"butterfly peak {pk.value/1e9:.1f} G/s")
for thr in (0, 4096):
  L.hc_set_cluster_threshold(thr)
  print("cluster threshold", thr)
  for dirn in (0, 1):
    for nj in (1, 2, 14, 16, 32, 148, 296, 592):
        us = ctypes.c_double()
        _lib.check(L.hc_bench_xform(h, nj, dirn, 50, ctypes.byref(us)))
        bf = nj * 4096 * 13 / (us.value * 1e-6) / 1e9
        print(f"  dir {dirn} jobs {nj:5d}: {us.value:8.2f} us/launch  {bf:7.1f} Gbfly/s")
L.hc_set_cluster_threshold(16)

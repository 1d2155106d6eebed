"""Transform microbenchmark / ncu driver: `njobs` independent 8192-point
NTTs (dir 0) or INTTs (dir 1) per launch (hc_bench_xform; >= 200 jobs run
the 256-thread three-per-SM variant k_xf<.., 4>).

  python tools/xform_bench.py [dir] [njobs] [iters]
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_17063_b200 as P
from paper_2408_17063_b200 import _lib

d = int(sys.argv[1]) if len(sys.argv) > 1 else 0
nj = int(sys.argv[2]) if len(sys.argv) > 2 else 592
it = int(sys.argv[3]) if len(sys.argv) > 3 else 3
be = P.B200BgvBackend(P.HeParams(8192, 65537, 3), seed=0)
L = _lib.lib()
h = be._ctx()
L.hc_set_cluster_threshold(0)
us = ctypes.c_double()
_lib.check(L.hc_bench_xform(h, nj, d, it, ctypes.byref(us)))
print(f"{nj} {'INTT' if d else 'NTT'}s per launch: {us.value:.2f} us, {nj * 53248 / (us.value * 1e-6) / 1e9:.1f} G butterflies/s")

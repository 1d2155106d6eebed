import os, sys, ctypes
sys.path.insert(0, os.getcwd())
import paper_2408_17063_b200 as P
from paper_2408_17063_b200 import _lib
be = P.B200BgvBackend(P.HeParams(8192, 65537, 3), seed=0)
L = _lib.lib(); h = be._ctx()
L.hc_set_cluster_threshold(0)
us = ctypes.c_double()
_lib.check(L.hc_bench_xform(h, 592, int(sys.argv[1]), 3, ctypes.byref(us)))
print(us.value)

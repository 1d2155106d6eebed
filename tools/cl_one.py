"""Run a few single-job cluster transforms (for ncu)."""
import os, sys, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_17063_b200 as P
from paper_2408_17063_b200 import _lib
be = P.B200BgvBackend(P.HeParams(8192, 65537, 3), seed=0)
L = _lib.lib(); h = be._ctx()
us = ctypes.c_double()
for d in (0, 1):
    _lib.check(L.hc_bench_xform(h, 2, d, 5, ctypes.byref(us)))
    print(d, us.value)

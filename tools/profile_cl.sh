#!/bin/bash
# Full ncu capture of the latency-path transforms inside bench.py's timed region:
# the fold digit NTT (k_xf_cl<0,5,6,1>), the fold two-prime INTT (k_cl16_intt2<8>)
# and the lane diagonal INTT (k_xf<1,1,5,1>).
O=gpurun_out
NCU=/usr/local/cuda/bin/ncu
$NCU --set full --import-source on --clock-control none --nvtx --nvtx-include "timed/" --kernel-name-base demangled \
  -k "regex:k_xf_cl<.int.0, .int.5, .int.6, .int.1>" --launch-skip 3 -c 1 -o $O/ncu_full_xf_cl_fold -f \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_full_cl.log 2>&1
$NCU --set full --import-source on --clock-control none --nvtx --nvtx-include "timed/" --kernel-name-base demangled \
  -k "regex:k_cl16_intt2<.int.8>" --launch-skip 3 -c 1 -o $O/ncu_full_intt2_fold -f \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_full_i2.log 2>&1
$NCU --set full --import-source on --clock-control none --nvtx --nvtx-include "timed/" --kernel-name-base demangled \
  -k "regex:k_xf<.int.1, .int.1, .int.5, .int.1>" --launch-skip 1 -c 1 -o $O/ncu_full_xf_diag_intt -f \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_full_dg.log 2>&1
ls -la $O/*.ncu-rep; for f in $O/ncu_full_cl.log $O/ncu_full_i2.log $O/ncu_full_dg.log; do tail -n 2 $f; done

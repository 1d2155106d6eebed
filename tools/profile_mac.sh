#!/bin/bash
# Full ncu capture of the throughput-regime MAC kernels at N=2^20, s=16
O=gpurun_out
NCU=/usr/local/cuda/bin/ncu
$NCU --set full --import-source on --clock-control none --nvtx --nvtx-include "timed/" --kernel-name-base demangled \
  -k "regex:k_ksmac" --launch-skip 1 -c 1 -o $O/ncu_full_ksmac_2e20 -f \
  python bench.py --N 1048576 --s 16 --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_mac.log 2>&1
$NCU --set full --import-source on --clock-control none --nvtx --nvtx-include "timed/" --kernel-name-base demangled \
  -k "regex:k_diagx" --launch-skip 1 -c 1 -o $O/ncu_full_diagx_2e20 -f \
  python bench.py --N 1048576 --s 16 --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_dx.log 2>&1
ls -la $O/*2e20*.ncu-rep

#!/bin/bash
# Round evidence on one B200 (run from the repo root under gpurun):
#   bench line + reference-arm line, launch list of the timed region (ncu,
#   gpu__time_duration only), full captures of the top transform kernels.
# Numbers taken under ncu are cold/serialised: shares, not absolutes.
set -x
O=gpurun_out
python bench.py > $O/bench_line.json 2> $O/bench.err; tail -1 $O/bench_line.json
python bench.py --impl reference --steps 3 --warmup 1 > $O/ref_line.json 2> $O/ref.err; tail -1 $O/ref_line.json
NCU=/usr/local/cuda/bin/ncu
$NCU --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
python tools/launch_table.py $O/launches.csv > $O/launches.txt; tail -14 $O/launches.txt
# throughput transform (592 jobs, VT=4) and the latency-path cluster digit NTT (fold, 14 jobs)
$NCU --set full --import-source on --clock-control none -k regex:k_xf -c 1 -o $O/ncu_full_xf_vt4 -f \
  python tools/nb1.py 0 > $O/ncu_full1.log 2>&1
$NCU --set full --import-source on --clock-control none --nvtx --nvtx-include "timed/" -k regex:k_xf_cl \
  --launch-skip 30 -c 1 -o $O/ncu_full_xf_cl -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_full2.log 2>&1
ls -la $O/*.ncu-rep

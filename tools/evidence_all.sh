#!/bin/bash
# Full round evidence on one B200; keeps gpurun_out/ small (ncu reports are
# summarised on the box and removed).
O=gpurun_out
bash tools/profile_r02.sh > $O/pr.log 2>&1
bash tools/profile_cl.sh > $O/pc.log 2>&1
bash tools/profile_mac.sh > $O/pm.log 2>&1
python tools/sweep.py 8192:8 16384:8 16384:16 16384:32 16384:64 16384:128 8192:16 32768:16 65536:16 131072:16 65536:64 1048576:16 1048576:128 4194304:16 4194304:128 > $O/sweep.txt 2>&1
python tools/sweep.py 16384:16 65536:64 1048576:16 --flush > $O/sweep_flush.txt 2>&1
python tools/trace_comp.py > $O/trace.txt 2>&1
python bench.py --N 1048576 --s 16 --steps 5 --warmup 3 > $O/bench_2e20.json 2>/dev/null
python tools/multi_query.py --Q 8 > $O/mq.txt 2>&1
(python tools/answer_bench.py --N 8192 --s 8; python tools/answer_bench.py --N 16384 --s 16; python tools/answer_bench.py --N 65536 --s 64) > $O/answer_bench.jsonl 2>&1
python tools/ncu_summary.py $O/ncu_full_xf_vt4.ncu-rep $O/ncu_full_xf_cl_fold.ncu-rep $O/ncu_full_intt2_fold.ncu-rep \
  $O/ncu_full_xf_diag_intt.ncu-rep $O/ncu_full_ksmac_2e20.ncu-rep $O/ncu_full_diagx_2e20.ncu-rep > $O/ncu_summary.txt 2>&1
for r in xf_vt4 xf_cl_fold intt2_fold xf_diag_intt ksmac_2e20 diagx_2e20; do
  ncu -i $O/ncu_full_$r.ncu-rep --page details --csv > $O/ncu_full_${r}_details.csv 2>/dev/null
done
rm -f $O/*.ncu-rep
tail -1 $O/bench_line.json | cut -c1-200

#!/bin/bash
# Round-2 ncu evidence on one B200 (run from the repo root under gpurun; one
# process at a time -- ncu replays each captured kernel ~40 times).  Numbers
# taken under ncu are cold-cache and serialised: compare shares, not absolutes.
#   1. launch list of bench.py's timed region (gpu__time_duration only)
#   2. ncu --set full of the headline's kernels inside the timed region and of
#      the N = 2^20 MAC kernels; summaries + details CSVs
#   3. DRAM bytes per launch of the dominant transform kernel -> the bench
#      line's roofline.traffic (profiles/r02_ncu_dominant_traffic.json)
O=gpurun_out/ncu
mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-parity"
if [ -z "$ONLY" ]; then
$NCU --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-parity > $O/launch.log 2>&1
python tools/launch_table.py $O/launches.csv > $O/launches.txt 2>&1
fi
cap() {  # name regex skip [cmd...]   (ONLY="a b": capture just those)
  local name=$1 rx=$2 skip=$3; shift 3
  if [ -n "$ONLY" ] && [[ " $ONLY " != *" $name "* ]]; then return; fi
  $NCU --set full --import-source on --clock-control none --nvtx --nvtx-include "timed/" --kernel-name-base demangled \
    -k "regex:$rx" --launch-skip $skip -c 1 -o $O/$name -f "$@" > $O/$name.log 2>&1
}
cap diag_intt   'k_xf<\(int\)1, \(int\)1, \(int\)5, \(int\)1>'       1 $B
cap foldchain   'k_foldchain'            0 $B
cap giant_ntt   'k_xf_cl<\(int\)0, \(int\)5, \(int\)6, \(int\)3>'    0 $B
cap ksmac_lat   'k_ksmac<\(int\)1, \(int\)4>'          1 $B
cap compose     'k_compose'              0 $B
cap pack_intt   'k_xf_cl<\(int\)1, \(int\)1, \(int\)9, \(int\)2>'    0 $B
cap ksmac_2e20  'k_ksmac_mb'             1 python bench.py --N 1048576 --sparsity 16 --steps 1 --warmup 3 --no-cpu-baseline --no-parity
cap diagx_2e20  'k_diagx'                1 python bench.py --N 1048576 --sparsity 16 --steps 1 --warmup 3 --no-cpu-baseline --no-parity
cap xf_dig_2e20 'k_xf<\(int\)0, \(int\)5, \(int\)7, \(int\)4>'       1 python bench.py --N 1048576 --sparsity 16 --steps 1 --warmup 3 --no-cpu-baseline --no-parity
cap diag_intt_2e20 'k_xf<\(int\)1, \(int\)1, \(int\)5, \(int\)4>'    1 python bench.py --N 1048576 --sparsity 16 --steps 1 --warmup 3 --no-cpu-baseline --no-parity
HC_KSFUSED=1 cap ksfused_2e20 'k_ksfused'  1 python bench.py --N 1048576 --sparsity 16 --steps 1 --warmup 3 --no-cpu-baseline --no-parity
[ -z "$ONLY" ] && $NCU --set full --import-source on --clock-control none -k 'regex:k_xf' -c 1 -o $O/xf_vt4 -f python tools/xform_bench.py 0 592 > $O/xf_vt4.log 2>&1
for r in diag_intt foldchain giant_ntt ksmac_lat compose pack_intt ksmac_2e20 diagx_2e20 xf_dig_2e20 diag_intt_2e20 ksfused_2e20 xf_vt4; do
  [ -f $O/$r.ncu-rep ] || continue
  $NCU -i $O/$r.ncu-rep --page details --csv > $O/${r}_details.csv 2>/dev/null
  $NCU -i $O/$r.ncu-rep --page raw --csv > $O/${r}_raw.csv 2>/dev/null
done
python tools/ncu_summary.py $O/*.ncu-rep > $O/summary.txt 2>&1
[ -f $O/diag_intt_raw.csv ] && python tools/ncu_traffic.py $O/diag_intt_raw.csv 'k_xf<1, 1, 5, 1>' 32 262144 > $O/traffic_diag_intt.json
# N = 2^20 (128-block chunks): 12672 digit NTTs per launch, each reads 8192 u16 digits + the u16 gather table and writes 64 KiB
[ -f $O/xf_dig_2e20_raw.csv ] && python tools/ncu_traffic.py $O/xf_dig_2e20_raw.csv 'k_xf<0, 5, 7, 4>' 12672 98304 > $O/traffic_xf_dig_2e20.json
[ -f $O/ksfused_2e20_raw.csv ] && python tools/ncu_traffic.py $O/ksfused_2e20_raw.csv 'k_ksfused' 384 646144 > $O/traffic_ksfused_2e20.json
python tools/ncu_stalls.py $O/ksfused_2e20.ncu-rep $O/xf_dig_2e20.ncu-rep $O/diag_intt_2e20.ncu-rep $O/foldchain.ncu-rep > $O/stalls.txt 2>&1
rm -f $O/*.ncu-rep
cat $O/summary.txt | head -80

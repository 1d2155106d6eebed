#!/bin/bash
# A/B of environment switches on the headline bench, alternating runs on one
# box:  bash tools/ab_env.sh "HC_FOLD_NCL=0" "HC_FOLD_NCL=13" [rounds]
# prints the median latency of each run (bench.py --no-cpu-baseline --no-parity)
A="$1"; B="$2"; R=${3:-3}; shift 3 2>/dev/null
for r in $(seq $R); do
  for v in "$A" "$B"; do
    ms=$(env $v python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-parity "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['latency_ms']['median'],4), round(d['e2e']['ms_per_step'],4))")
    echo "$v: median_ms e2e_ms = $ms"
  done
done

#!/bin/bash
# Headline A/B of an environment switch on one box: bash tools/env_ab.sh VAR [reps]
V=$1; R=${2:-3}
P='import json,sys; d=json.load(sys.stdin); print({k: round(x, 4) for k, x in d["latency_ms"].items()}, "e2e", round(d["e2e"]["value"]/1e6,2))'
for i in $(seq $R); do
  for v in 0 1; do echo -n "$V=$v: "; env $V=$v python bench.py --no-cpu-baseline 2>/dev/null | tail -1 | python -c "$P"; done
done

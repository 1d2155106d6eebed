#!/bin/bash
# GPU check used between kernel changes: parity tests, bench with/without PDL, trace.
# usage (on the GPU box): bash tools/gpu_quick.sh [tests=1] [trace=1]
T=${1:-1}; TR=${2:-1}
[ "$T" = 1 ] && python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for v in 1 0; do
  HC_PDL=$v python bench.py --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print('PDL', $v, 'lat ms', {k: round(x, 4) for k, x in d['latency_ms'].items()}, 'e2e M/s', round(d['e2e']['value']/1e6, 2))"
done
if [ "$TR" = 1 ]; then python tools/trace_comp.py > gpurun_out/trace.txt 2>&1; tail -1 gpurun_out/trace.txt; fi

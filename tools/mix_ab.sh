python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "reversed or answer or five_prime or below_level" 2>&1 | tail -2
P='import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    m=d["ms"]; print(d["workload"][38:62], "dev", m["answer_graph_device_resident (CUDA events, L2 flushed)"], "comp_mixed", m["comp_mixed"], "ans", m["answer_from_match"])'
for v in "HC_MIX_LANES=0" "HC_MIX_LANES=1" "HC_MIX_CL=0"; do
  echo "== $v"
  for pt in "8192 8" "16384 16" "65536 64"; do set -- $pt; env $v python tools/answer_bench.py --N $1 --s $2 2>/dev/null | python -c "$P"; done
done

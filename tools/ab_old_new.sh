# A/B: old (worktree) vs new, alternating on one box
B="python bench.py --no-cpu-baseline"
P='import json,sys; d=json.load(sys.stdin); print({k: round(x, 4) for k, x in d["latency_ms"].items()}, "e2e", round(d["e2e"]["value"]/1e6,2))'
for i in 1 2 3; do
  echo -n "old: "; (cd _ab_old && $B 2>/dev/null | tail -1 | python -c "$P")
  echo -n "new: "; ($B 2>/dev/null | tail -1 | python -c "$P")
done

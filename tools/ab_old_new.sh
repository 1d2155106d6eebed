# A/B(/C): old (worktree _ab_old) vs new, alternating on one box; variant C =
# this tree's code built with -DHC_MAXL=3 into _ab_c/ (when present)
B="python bench.py --no-cpu-baseline"
P='import json,sys; d=json.load(sys.stdin); print({k: round(x, 4) for k, x in d["latency_ms"].items()}, "e2e", round(d["e2e"]["value"]/1e6,2))'
for i in 1 2 3; do
  echo -n "old: "; (cd _ab_old && $B 2>/dev/null | tail -1 | python -c "$P")
  echo -n "new: "; ($B 2>/dev/null | tail -1 | python -c "$P")
  if [ -f _ab_c/libhcomp.so ]; then echo -n "C:   "; (HCOMP_LIB=$PWD/_ab_c/libhcomp.so $B 2>/dev/null | tail -1 | python -c "$P"); fi
done

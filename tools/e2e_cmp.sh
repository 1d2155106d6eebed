for f in 1 0; do
  python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-flush $f 2>/dev/null | tail -1 > gpurun_out/b$f.json
  python3 -c "import json,sys; d=json.load(open('gpurun_out/b$f.json')); print('flush $f', d['ms_per_step'], d['e2e']['ms_per_step'], d['e2e']['serial_ms_per_step'])"
done

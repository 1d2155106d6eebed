python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -2 gpurun_out/gpu_tests.log
rm -f gpurun_out/config4_oracle.jsonl
for pt in "1048576 16" "1048576 128" "4194304 16" "4194304 128"; do
  set -- $pt
  timeout 1500 python tools/large_config.py --N $1 --s $2 --iters 5 --oracle --json gpurun_out/config4_oracle.jsonl > /dev/null 2>> gpurun_out/config4_oracle.err; echo "N=$1 s=$2 rc=$?"
done
timeout 900 python tools/multi_query.py --Q 8 --oracle 4 > gpurun_out/config5_oracle.txt 2>&1; echo "multi rc=$?"; tail -3 gpurun_out/config5_oracle.txt
nproc; lscpu | grep "Model name"

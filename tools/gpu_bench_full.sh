timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_default.log
for c in 64 74 96; do
  timeout 400 python bench.py --ctas-per-chain $c --no-cpu-baseline --no-e2e > gpurun_out/bench_c8_$c.log 2>&1; echo "c8 ctas=$c rc=$?"
  tail -1 gpurun_out/bench_c8_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', round(d['value'],2), 'it', round(d['iterations_mean'],1), 'split', d['time_split_ms'])"
done
timeout 400 python bench.py --chains 16 --no-cpu-baseline --no-e2e > gpurun_out/bench_c16.log 2>&1; echo "c16 rc=$?"
tail -1 gpurun_out/bench_c16.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', round(d['value'],2), 'it', round(d['iterations_mean'],1), 'split', d['time_split_ms'])"

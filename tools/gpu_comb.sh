timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
timeout 300 python tools/prof_big.py 4 2 > gpurun_out/big4.log 2>&1; echo "C4 rc=$?"; tail -1 gpurun_out/big4.log | cut -c150-400
for i in 1 2; do
timeout 400 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_$i.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench_$i.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', round(d['value'],2), 'it', round(d['iterations_mean'],1), 'split', d['time_split_ms'], 'agg', round(d['roofline']['aggregate_gbs']))"
done
timeout 400 python bench.py --chains 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_1c.log 2>&1; echo "bench 1 chain rc=$?"
tail -1 gpurun_out/bench_1c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', round(d['value'],2), 'it', round(d['iterations_mean'],1), 'split', d['time_split_ms'], 'roof', round(d['roofline']['achieved']))"

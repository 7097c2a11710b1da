timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
timeout 300 python tools/prof_dense.py > gpurun_out/prof_dense.log 2>&1; echo "prof_dense rc=$?"; head -20 gpurun_out/prof_dense.log
timeout 400 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_default.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench_default.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', round(d['value'],2), 'it', round(d['iterations_mean'],1), 'split', d['time_split_ms'])"
timeout 400 python bench.py --chains 4 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4.log 2>&1; echo "bench c4 rc=$?"
tail -1 gpurun_out/bench_c4.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', round(d['value'],2), 'it', round(d['iterations_mean'],1), 'split', d['time_split_ms'], d['config']['ctas_per_chain'])"

timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for tm in 1 0; do
  if [ $tm = 0 ]; then export SKR_NO_TMA=1; fi
  timeout 300 python tools/prof_big.py 4 2 > gpurun_out/big4_t$tm.log 2>&1; echo "C4 tma=$tm rc=$?"; tail -1 gpurun_out/big4_t$tm.log | cut -c150-400
  timeout 300 python tools/prof_big.py 3 1 > gpurun_out/big3_t$tm.log 2>&1; echo "C3 tma=$tm rc=$?"; tail -1 gpurun_out/big3_t$tm.log | cut -c150-400
  timeout 400 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_t$tm.log 2>&1; echo "bench tma=$tm rc=$?"
  tail -1 gpurun_out/bench_t$tm.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', round(d['value'],2), 'it', round(d['iterations_mean'],1), 'split', d['time_split_ms'], 'agg', round(d['roofline']['aggregate_gbs']))"
done
unset SKR_NO_TMA
SKR_NO_CSR_CACHE=1 timeout 400 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_nocsr.log 2>&1; echo "bench nocsr rc=$?"
tail -1 gpurun_out/bench_nocsr.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', round(d['value'],2), 'it', round(d['iterations_mean'],1), 'split', d['time_split_ms'], 'agg', round(d['roofline']['aggregate_gbs']))"
timeout 300 python tools/prof_dense.py > gpurun_out/prof_dense.log 2>&1; echo "prof_dense rc=$?"; grep "cycle_ms\|cycle sweep\|barrier" gpurun_out/prof_dense.log

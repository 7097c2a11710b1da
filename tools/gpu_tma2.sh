timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
big() { tag=$1; shift; env "$@" timeout 300 python tools/prof_big.py 4 2 > gpurun_out/big4_$tag.log 2>&1; echo "C4 $tag rc=$?"; tail -1 gpurun_out/big4_$tag.log | cut -c150-400; }
big tma
big notma SKR_NO_TMA=1
big notma_co100 SKR_NO_TMA=1 SKR_CARVEOUT=100
big tma_co100 SKR_CARVEOUT=100
timeout 300 python tools/prof_big.py 3 1 > gpurun_out/big3.log 2>&1; echo "C3 tma rc=$?"; tail -1 gpurun_out/big3.log | cut -c150-400
for tm in 1 0; do
  if [ $tm = 0 ]; then export SKR_NO_TMA=1; fi
  timeout 400 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_t$tm.log 2>&1; echo "bench tma=$tm rc=$?"
  tail -1 gpurun_out/bench_t$tm.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', round(d['value'],2), 'it', round(d['iterations_mean'],1), 'split', d['time_split_ms'], 'agg', round(d['roofline']['aggregate_gbs']))"
done

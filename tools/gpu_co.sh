timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
big() { tag=$1; shift; env "$@" timeout 300 python tools/prof_big.py 4 2 > gpurun_out/big4_$tag.log 2>&1; echo "C4 $tag rc=$?"; tail -1 gpurun_out/big4_$tag.log | cut -c200-400; }
big def
big co25 SKR_CARVEOUT=25
big co50 SKR_CARVEOUT=50
big co64 SKR_CARVEOUT=64
big co80 SKR_CARVEOUT=80
for co in def 64; do
  if [ $co = def ]; then unset SKR_CARVEOUT; else export SKR_CARVEOUT=$co; fi
  timeout 400 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_co$co.log 2>&1; echo "bench co=$co rc=$?"
  tail -1 gpurun_out/bench_co$co.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', round(d['value'],2), 'it', round(d['iterations_mean'],1), 'split', d['time_split_ms'], 'agg', round(d['roofline']['aggregate_gbs']))"
done

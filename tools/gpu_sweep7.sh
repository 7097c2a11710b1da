timeout 300 python tools/prof_dense.py > gpurun_out/prof_dense.log 2>&1; echo "prof_dense rc=$?"; grep "hqr\|LU" gpurun_out/prof_dense.log
for cfg in "2 148" "2 296" "4 74" "4 100" "8 48" "8 64"; do
  set -- $cfg
  timeout 400 python bench.py --chains $1 --ctas-per-chain $2 --no-cpu-baseline --no-e2e > gpurun_out/bench_c$1_$2.log 2>&1; echo "chains=$1 ctas=$2 rc=$?"
  tail -1 gpurun_out/bench_c$1_$2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', round(d['value'],2), 'it', round(d['iterations_mean'],1), 'split', d['time_split_ms'], 'agg', round(d['roofline']['aggregate_gbs']))"
done

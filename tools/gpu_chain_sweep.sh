# chains x CTAs-per-chain sweep of the default C1 bench (no e2e / cpu legs)
for cfg in ${SWEEP:-"8 64" "8 37" "10 29" "12 24" "16 18" "12 36" "16 27"}; do
  set -- $cfg
  timeout 400 python bench.py --no-cpu-baseline --no-e2e --chains $1 --ctas-per-chain $2 --stripe $((2 * $1)) > gpurun_out/sweep_$1_$2.log 2>&1
  echo -n "chains=$1 ctas=$2 rc=$? "
  tail -1 gpurun_out/sweep_$1_$2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', round(d['value'],2), 'it', round(d['iterations_mean'],1), 'agg', round(d['roofline']['aggregate_gbs']))"
done

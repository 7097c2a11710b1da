for cfg in "8 64" "4 74" "4 100" "8 48" "8 56" "8 80" "16 32" "8 64"; do
  set -- $cfg
  timeout 400 python bench.py --chains $1 --ctas-per-chain $2 --no-cpu-baseline --no-e2e > gpurun_out/sw_$1_$2.log 2>&1; echo "chains=$1 ctas=$2 rc=$?"
  tail -1 gpurun_out/sw_$1_$2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', round(d['value'],2), 'it', round(d['iterations_mean'],1), 'roof', round(d['roofline']['achieved']))"
done

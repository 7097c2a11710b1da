for sh in "8 37 8" "9 37 9" "10 37 10" "10 33 10" "12 30 12" "9 33 9" "16 20 16" "8 37 16"; do
  set -- $sh
  timeout 400 python bench.py --config 3 --chains $1 --ctas-per-chain $2 --stripe $3 --no-cpu-baseline --no-e2e > gpurun_out/sw_$1_$2_$3.log 2>&1
  tail -1 gpurun_out/sw_$1_$2_$3.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C3 chains $1 x $2 stripe $3: value', round(d['value'],3), 'it', round(d['iterations_mean'],2), d['all_converged'], 'dense ms', round(d['time_split_ms']['dense_recycle_kernels']), 'cyc', round(d['time_split_ms']['cycle_kernels']), 'tot', round(d['time_split_ms']['total']))"
done

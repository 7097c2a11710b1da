# A/B of the working-tree build against alt/$ALT: bench C1 and C3 (device pass only), twice each
ALT=${ALT:-prev}
for v in $ALT cur $ALT cur; do
  if [ $v = cur ]; then unset SKR_LIB_PATH; else export SKR_LIB_PATH=$PWD/alt/$v/libskr.so; fi
  for c in ${CFGS:-1 3}; do
  timeout 400 python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/ab_${c}_$v.log 2>&1
  tail -1 gpurun_out/ab_${c}_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C$c $v value', round(d['value'],3), 'it', round(d['iterations_mean'],2), d['all_converged'], 'agg', round(d['roofline']['aggregate_gbs']), 'split', {k: round(v) for k, v in d['time_split_ms'].items() if k != 'chain_wall_ms'})"
  done
done

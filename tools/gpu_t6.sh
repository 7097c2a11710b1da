timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
for v in fuse1 cur prev cur; do
  if [ $v = cur ]; then unset SKR_LIB_PATH; else export SKR_LIB_PATH=$PWD/alt/$v/libskr.so; fi
  for c in 1 3; do
  timeout 400 python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/ab_${c}_$v.log 2>&1
  tail -1 gpurun_out/ab_${c}_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C$c $v value', round(d['value'],3), 'it', round(d['iterations_mean'],2), d['all_converged'])"
  done
done
unset SKR_LIB_PATH
for sh in "4 74 8" "6 49 12" "8 37 8" "12 24 12" "12 48 12" "16 32 16"; do
  set -- $sh
  timeout 400 python bench.py --config 3 --chains $1 --ctas-per-chain $2 --stripe $3 --no-cpu-baseline --no-e2e > gpurun_out/sw_$1_$2.log 2>&1
  tail -1 gpurun_out/sw_$1_$2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C3 chains $1 x $2 stripe $3: value', round(d['value'],3), 'it', round(d['iterations_mean'],2), d['all_converged'])"
done

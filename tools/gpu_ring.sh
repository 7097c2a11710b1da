timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "chain or c3_eight or collect" > gpurun_out/pt.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pt.log
for v in regpf cur ring3 regpf cur ring3; do
  if [ $v = cur ]; then unset SKR_LIB_PATH; else export SKR_LIB_PATH=$PWD/alt/$v/libskr.so; fi
  timeout 400 python bench.py --config 3 --no-cpu-baseline --no-e2e > gpurun_out/r_$v.log 2>&1
  tail -1 gpurun_out/r_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C3 $v value', round(d['value'],3), 'it', round(d['iterations_mean'],2), d['all_converged'])"
done
unset SKR_LIB_PATH
timeout 600 python tools/prof_chains.py 3 16 8 37 2>&1 | grep "all chains"

timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for i in 1 2 3; do timeout 900 python tools/c3_chains_probe.py 3 16 8 > gpurun_out/c3probe_$i.log 2>&1; echo "c3probe $i rc=$?"; grep chunk gpurun_out/c3probe_$i.log; done
SKR_LIB_PATH=$PWD/alt/diag/libskr.so timeout 900 python tools/c3_chains_probe.py 3 16 8 > gpurun_out/diag2_c3.log 2>&1
SKR_LIB_PATH=$PWD/alt/diag/libskr.so timeout 900 python tools/c3_chains_probe.py 4 4 2 > gpurun_out/diag2_c4.log 2>&1
SKR_LIB_PATH=$PWD/alt/diag/libskr.so timeout 900 python tools/c3_chains_probe.py 2 8 4 > gpurun_out/diag2_c2.log 2>&1; grep chunk gpurun_out/diag2_c2.log
for v in base cur base cur; do
  if [ $v = cur ]; then unset SKR_LIB_PATH; else export SKR_LIB_PATH=$PWD/alt/$v/libskr.so; fi
  timeout 400 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/abb_$v.log 2>&1; echo "bench $v rc=$?"
  tail -1 gpurun_out/abb_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', round(d['value'],2), 'split', d['time_split_ms'])"
done

timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for i in 1 2 3; do timeout 600 python tools/c3_chains_probe.py 3 16 8 > gpurun_out/det_c3_$i.log 2>&1; grep chunk gpurun_out/det_c3_$i.log | md5sum; done
grep chunk gpurun_out/det_c3_1.log | head -3
for i in 1 2 3; do timeout 600 python tools/c3_chains_probe.py 4 4 2 > gpurun_out/det_c4_$i.log 2>&1; grep chunk gpurun_out/det_c4_$i.log; done
for i in 1 2 3; do timeout 600 python tools/c3_chains_probe.py 1 32 8 > gpurun_out/det_c1_$i.log 2>&1; grep chunk gpurun_out/det_c1_$i.log | md5sum; done
for v in prev cur prev cur; do
  if [ $v = cur ]; then unset SKR_LIB_PATH; else export SKR_LIB_PATH=$PWD/alt/$v/libskr.so; fi
  timeout 400 python bench.py --config 1 --no-cpu-baseline --no-e2e > gpurun_out/abb_$v.log 2>&1; echo "bench c1 $v rc=$?"
  tail -1 gpurun_out/abb_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', round(d['value'],2), 'it', d['iterations_mean'])"
  timeout 400 python bench.py --config 3 --no-cpu-baseline --no-e2e > gpurun_out/abb3_$v.log 2>&1; echo "bench c3 $v rc=$?"
  tail -1 gpurun_out/abb3_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', round(d['value'],3), 'it', d['iterations_mean'], d['all_converged'])"
done

for v in cur bprev cur bprev; do
  if [ $v = cur ]; then unset SKR_LIB_PATH; else export SKR_LIB_PATH=$PWD/alt/$v/libskr.so; fi
  timeout 300 python tools/prof_dense.py > gpurun_out/abd_$v.log 2>&1; echo "dense $v rc=$?"; grep "cycle_ms\|barrier\|resid" gpurun_out/abd_$v.log | head -6
  timeout 400 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/abb_$v.log 2>&1; echo "bench $v rc=$?"
  tail -1 gpurun_out/abb_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', round(d['value'],2), 'split', d['time_split_ms'])"
done
timeout 300 python tools/prof_big.py 4 2 > gpurun_out/ab_c4.log 2>&1; echo "C4 cur rc=$?"; tail -1 gpurun_out/ab_c4.log | cut -c200-400
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log

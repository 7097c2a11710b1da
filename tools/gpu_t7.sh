timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
for v in prev cur; do
  if [ $v = cur ]; then unset SKR_LIB_PATH; else export SKR_LIB_PATH=$PWD/alt/$v/libskr.so; fi
  timeout 400 python bench.py --config 1 --no-cpu-baseline --no-e2e > gpurun_out/ab_1_$v.log 2>&1
  tail -1 gpurun_out/ab_1_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C1 $v value', round(d['value'],3), 'it', round(d['iterations_mean'],2), d['all_converged'])"
done
unset SKR_LIB_PATH
for f in 0 1; do SKR_FUSE_COMB=$f timeout 400 python bench.py --config 3 --no-cpu-baseline --no-e2e > gpurun_out/fc_$f.log 2>&1
  tail -1 gpurun_out/fc_$f.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C3 fuse $f value', round(d['value'],3), 'it', round(d['iterations_mean'],2), d['all_converged'], d['config']['ctas_per_chain'])"; done
for sh in "8 37 8" "8 64 8" "4 74 8" "2 148 4"; do
  set -- $sh
  timeout 600 python bench.py --config 4 --chains $1 --ctas-per-chain $2 --stripe $3 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/sw4_$1_$2.log 2>&1
  tail -1 gpurun_out/sw4_$1_$2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C4 chains $1 x $2: value', round(d['value'],3), 'it', round(d['iterations_mean'],2), d['all_converged'], 'gen', d['sort'])"
done
timeout 900 python bench.py > gpurun_out/bench_c3.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_c3.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k: d[k] for k in ('value','e2e','all_converged','iterations_mean','roofline','cpu_baseline','clocks','gpu_launches')})"

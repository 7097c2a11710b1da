timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
timeout 300 python tools/prof_big.py 4 2 > gpurun_out/big4.log 2>&1; echo "C4 rc=$?"; tail -1 gpurun_out/big4.log | cut -c1-400
timeout 400 python tools/prof_big.py 3 1 > gpurun_out/big3.log 2>&1; echo "C3 rc=$?"; tail -1 gpurun_out/big3.log | cut -c1-400
timeout 300 python tools/prof_dense.py > gpurun_out/prof_dense.log 2>&1; echo "prof_dense rc=$?"; grep "cycle" gpurun_out/prof_dense.log
run() {  # name, env..., args
  name=$1; shift
  env "$@" timeout 400 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e $BARGS > gpurun_out/bench_$name.log 2>&1; echo "$name rc=$?"
  tail -1 gpurun_out/bench_$name.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', round(d['value'],2), 'it', round(d['iterations_mean'],1), 'split', d['time_split_ms'], 'us/step', round(d['us_per_arnoldi_step'],2), 'roof', d['roofline']['achieved'])" 2>&1 | tail -1
}
BARGS="--chains 1" run c1
BARGS="--chains 8 --free-sms 8" run c8f8
BARGS="--chains 8 --free-sms 0" run c8n18 SKR_NBLK=18
BARGS="--chains 16 --free-sms 0" run c16n36 SKR_NBLK=36
BARGS="--chains 8 --free-sms 0" run c8n36 SKR_NBLK=36

run() {  # name, env..., args
  name=$1; shift
  env "$@" timeout 400 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e $BARGS > gpurun_out/bench_$name.log 2>&1; echo "$name rc=$?"
  tail -1 gpurun_out/bench_$name.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', round(d['value'],2), 'it', round(d['iterations_mean'],1), 'split', d['time_split_ms'], 'us/step', round(d['us_per_arnoldi_step'],2), 'roof', d['roofline']['achieved'])" 2>&1 | tail -1
}
BARGS="--chains 8 --free-sms 0" run c8n96 SKR_NBLK=96
BARGS="--chains 8 --free-sms 0" run c8n128 SKR_NBLK=128
BARGS="--chains 8 --free-sms 0" run c8n148 SKR_NBLK=148
BARGS="--chains 16 --free-sms 0" run c16n72 SKR_NBLK=72
BARGS="--chains 16 --free-sms 0" run c16n96 SKR_NBLK=96
BARGS="--chains 8 --free-sms 0" run c8n60 SKR_NBLK=60
BARGS="--chains 8 --free-sms 0" run c8n72r1 SKR_NBLK=72 SKR_CYCLE_R=1

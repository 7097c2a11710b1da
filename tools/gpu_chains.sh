for nc in 1 2 4; do
  timeout 900 python bench.py --chains $nc --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_chains_$nc.log 2>&1; echo "chains=$nc rc=$?"
  tail -1 gpurun_out/bench_chains_$nc.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', round(d['value'],2), 'it', round(d['iterations_mean'],1), 'split', d['time_split_ms'], 'us/step', round(d['us_per_arnoldi_step'],2))"
done

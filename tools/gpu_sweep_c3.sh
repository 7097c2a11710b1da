# chain-shape sweep at the HBM-gated configs (C3, C4) with the current bench
nproc; free -g | head -2
for c in 8 4 2 1; do
  S=$((c*2)); [ $c -ge 4 ] && S=$c
  timeout 900 python bench.py --config 3 --chains $c --stripe $S --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/sw3_$c.log 2>&1; echo "C3 chains $c rc=$?"
  tail -1 gpurun_out/sw3_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', round(d['value'],3), 'it', round(d['iterations_mean'],1), 'conv', d['all_converged'], 'roof', round(d['roofline']['aggregate_gbs']), round(d['roofline']['per_launch_gbs']), 'split', d['time_split_ms']['cycle_kernels'], d['time_split_ms']['dense_recycle_kernels'], d['time_split_ms']['total'], 'sort', d['sort'])"
done
for c in 8 4 2 1; do
  S=$c
  timeout 900 python bench.py --config 4 --n-systems 256 --chains $c --stripe $S --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/sw4_$c.log 2>&1; echo "C4 chains $c rc=$?"
  tail -1 gpurun_out/sw4_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', round(d['value'],3), 'it', round(d['iterations_mean'],1), 'conv', d['all_converged'], 'roof', round(d['roofline']['aggregate_gbs']), round(d['roofline']['per_launch_gbs']), 'split', d['time_split_ms']['cycle_kernels'], d['time_split_ms']['dense_recycle_kernels'], d['time_split_ms']['total'], 'sort', d['sort'])"
done

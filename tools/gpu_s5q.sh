timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
run() { timeout 600 python bench.py --config 3 --no-cpu-baseline --no-e2e --gen device 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['value'],3), 'it', round(d['iterations_mean'],2), d['all_converged'], 'split', {k: round(v) for k, v in d['time_split_ms'].items() if k != 'chain_wall_ms'})"; }
for rep in 1 2; do
unset SKR_GRAM_SIMPLE; run gram_dmma
export SKR_GRAM_SIMPLE=1; run gram_simple; unset SKR_GRAM_SIMPLE
done
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu launch rc=$?"
python tools/launch_summary.py /tmp/launches.csv | head -12

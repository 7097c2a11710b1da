for S in 8 16; do
timeout 900 python bench.py --config 3 --no-cpu-baseline --no-e2e --gen device --stripe $S 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('stripe $S', round(d['value'],3), 'it', round(d['iterations_mean'],2), d['all_converged'], round(d['ms_per_step'],1))"
done

timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
timeout 900 python tools/prof_precond.py 1 3 2>&1 | grep -v Warn
timeout 900 python tools/prof_precond.py 3 2 2>&1 | grep -v Warn
timeout 600 python bench.py --config 3 --no-cpu-baseline --no-e2e --gen device 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench C3', round(d['value'],3), 'it', round(d['iterations_mean'],2), d['all_converged'])"

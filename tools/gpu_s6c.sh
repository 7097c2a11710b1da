timeout 900 python -m pytest tests/test_precond.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
timeout 900 python tools/prof_precond.py 1 3 2>&1 | grep -v Warn
timeout 900 python tools/prof_precond.py 3 2 2>&1 | grep -v Warn

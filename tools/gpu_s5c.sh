timeout 900 python -m pytest tests/test_precond.py -m gpu -x -q -s -p no:cacheprovider 2>&1 | grep -v Warn | tail -40

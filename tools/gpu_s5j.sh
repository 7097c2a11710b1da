timeout 900 python -m pytest tests/test_precond.py -m gpu -x -q -p no:cacheprovider -k "side_paths" 2>&1 | grep -v Warn | tail -30

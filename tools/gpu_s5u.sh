timeout 900 python -m pytest tests/test_precond.py -m gpu -x -q -p no:cacheprovider -k "general_csr" 2>&1 | tail -25

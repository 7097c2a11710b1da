timeout 900 python -m pytest tests/test_precond.py tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -4

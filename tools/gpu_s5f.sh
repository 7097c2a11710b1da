timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -s -p no:cacheprovider -k "grouped or principal or sort" 2>&1 | grep -v Warn | tail -20

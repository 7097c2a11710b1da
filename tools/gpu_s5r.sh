timeout 900 python -m pytest tests/test_full_parity.py -k "prefix" -q -s -p no:cacheprovider 2>&1 | grep -E "gpu \[|passed|failed"

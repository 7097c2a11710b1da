# session 5: cycle-start profile points, half-Gram A/B (8-chain C3 shape) + full-size parity with it
for H in 0 1; do
echo "== SKR_GRAM_HALF=$H"
SKR_GRAM_HALF=$H timeout 600 python tools/prof_chains.py 3 16 8 37 2>&1 | grep -v Warn
done
SKR_GRAM_HALF=1 timeout 1500 python -m pytest tests/test_full_parity.py -k "prefix or c0_full" -q -s -p no:cacheprovider 2>&1 | grep -v Warn | tail -15

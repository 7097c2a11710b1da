# R (rows per lane) A/B in the 8-chain C3 bench shape
for R in 4 2; do
echo "== SKR_CYCLE_R=$R"
SKR_CYCLE_R=$R timeout 600 python bench.py --no-cpu-baseline --no-e2e --gen device 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['all_converged'], d['iterations_mean'])"
done

# chain-count variants in the C3 bench (all co-resident: chains x CTAs <= 296)
for V in "10 29" "9 32" "6 49" "8 37"; do
set -- $V
echo "== chains $1 x ctas $2"
timeout 900 python bench.py --no-cpu-baseline --no-e2e --gen device --chains $1 --ctas-per-chain $2 --stripe $1 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['all_converged'], d['iterations_mean'], d['ms_per_step'])"
done

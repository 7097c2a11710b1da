# C1: more chains so that the single-CTA dense updates overlap more sweeps
for V in "8 64" "12 48" "16 32" "16 18" "24 24"; do
set -- $V
echo "== chains $1 x ctas $2"
timeout 600 python bench.py --config 1 --no-cpu-baseline --no-e2e --chains $1 --ctas-per-chain $2 --stripe $1 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['value'],2), round(d['roofline']['frac'],3), d['all_converged'], round(d['iterations_mean'],1), {k: round(v) for k, v in d['time_split_ms'].items() if k != 'chain_wall_ms'})"
done

# every BASELINE config through the bench (device pass + cpu_baseline sample), for BASELINE.md section 4
for c in 0 1 2 4 3; do
  timeout 900 python bench.py --config $c > gpurun_out/all_$c.log 2>&1; echo "C$c rc=$?"
  tail -1 gpurun_out/all_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('C$c', 'value', round(d['value'],3), 'e2e', round(d['e2e']['value'],3) if d.get('e2e') else None, 'it', round(d['iterations_mean'],1), 'conv', d['all_converged'], 'agg', round(r['aggregate_gbs']), 'frac', round(r['frac'],3), 'cpu', d.get('cpu_baseline',{}).get('value'), d['config']['chains_per_gpu'], d['config']['ctas_per_chain'])"
done

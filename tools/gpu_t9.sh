for v in 1e-6 1e-9 1e-12; do
  SKR_V0_RTOL=$v timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k collect_diag > gpurun_out/pd_$v.log 2>&1; echo "diag $v rc=$?"; grep -E "^E  .*Assert" gpurun_out/pd_$v.log | head -2
  SKR_V0_RTOL=$v timeout 900 python -m pytest tests/test_full_parity.py -m gpu -q -s -k prefix > gpurun_out/pf_$v.log 2>&1; echo "full $v rc=$?"; grep -E "gpu \[" gpurun_out/pf_$v.log
  SKR_V0_RTOL=$v timeout 400 python bench.py --config 3 --no-cpu-baseline --no-e2e > gpurun_out/b3_$v.log 2>&1; tail -1 gpurun_out/b3_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C3 $v value', round(d['value'],3), 'it', round(d['iterations_mean'],2), d['all_converged'], d['v0_projected_cycles'])"
done

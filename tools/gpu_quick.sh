# Quick GPU check after a kernel change: parity tests, smoke(), dense/cycle
# phase profile (C1, one chain), C4 bandwidth (one chain), default bench x2.
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 300 python tools/prof_dense.py > gpurun_out/prof_dense.log 2>&1; echo "prof_dense rc=$?"; grep "cycle_ms\|hqr  \|cycle sweep\|barrier\|LS" gpurun_out/prof_dense.log
timeout 300 python tools/prof_big.py 4 2 > gpurun_out/quick_c4.log 2>&1; echo "C4 rc=$?"; tail -1 gpurun_out/quick_c4.log | cut -c200-400
for i in 1 2; do
  timeout 400 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/quick_b$i.log 2>&1; echo "bench rc=$?"
  tail -1 gpurun_out/quick_b$i.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', round(d['value'],2), 'it', round(d['iterations_mean'],1), 'split', d['time_split_ms'], 'agg', round(d['roofline']['aggregate_gbs']))"
done

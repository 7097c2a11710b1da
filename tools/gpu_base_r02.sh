# Round-2 baseline on the box: GPU tests, smoke, the C3 8-chain probe, C4 gate, default bench.
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python tools/c3_chains_probe.py 3 16 8 > gpurun_out/c3probe.log 2>&1; echo "c3probe rc=$?"; cat gpurun_out/c3probe.log | tail -10
timeout 400 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_c1.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_c1.log | cut -c1-600

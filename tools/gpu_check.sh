set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
tail -12 gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -40 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 2 --warmup 1 --stripe 4 --no-cpu-baseline > gpurun_out/bench_small.log 2>&1; echo bench_small_rc=$?
tail -20 gpurun_out/bench_small.log

timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_c3.log 2>&1; echo "bench c3 rc=$?"; tail -1 gpurun_out/bench_c3.log
timeout 900 python bench.py --impl reference > gpurun_out/bench_c3_ref.log 2>&1; echo "ref c3 rc=$?"; tail -1 gpurun_out/bench_c3_ref.log
timeout 600 python bench.py --config 1 --no-cpu-baseline > gpurun_out/bench_c1.log 2>&1; echo "bench c1 rc=$?"; tail -1 gpurun_out/bench_c1.log | cut -c1-300

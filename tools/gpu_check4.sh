timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python tools/prof_dense.py 1 2 2>&1 | grep -v "Warn\|return torch\|(at 1.9"
timeout 900 python tools/prof_big.py 4 1 2>&1 | tail -1
timeout 900 python tools/prof_big.py 3 2 2>&1 | tail -1

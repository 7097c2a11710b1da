timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python tools/prof_dense.py 1 2 > gpurun_out/prof_dense.log 2>&1; echo rc=$?
grep -v "Warn\|return torch" gpurun_out/prof_dense.log | grep -v "^  [a-zA-Z+()]* .*us/call"

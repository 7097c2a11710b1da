timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python tools/prof_dense.py 3 2 > gpurun_out/prof_c3.log 2>&1; echo rc=$?; grep -E "iterations|cycle" gpurun_out/prof_c3.log
ALT=prev bash tools/gpu_ab2.sh

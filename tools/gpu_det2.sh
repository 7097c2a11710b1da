timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
for i in 1 2; do timeout 600 python tools/c3_chains_probe.py 1 32 8 > gpurun_out/det_c1_$i.log 2>&1; grep chunk gpurun_out/det_c1_$i.log | md5sum; done
bash tools/gpu_ab2.sh

python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -4
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_final2.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu_final2.log

timeout 900 python -m pytest tests/test_grf.py -x -q -p no:cacheprovider > gpurun_out/pytest_grf.log 2>&1; echo "grf rc=$?"; tail -15 gpurun_out/pytest_grf.log
timeout 300 python tools/prof_dense.py 1 3 > gpurun_out/prof_dense_c1.log 2>&1; cat gpurun_out/prof_dense_c1.log
SKR_PROF_CTAS=37 timeout 600 python tools/prof_dense.py 3 2 > gpurun_out/prof_dense_c3.log 2>&1; cat gpurun_out/prof_dense_c3.log

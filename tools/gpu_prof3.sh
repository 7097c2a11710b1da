timeout 300 python tools/prof_dense.py 3 2 > gpurun_out/prof_c3.log 2>&1; echo rc=$?; cat gpurun_out/prof_c3.log
SKR_PROF_CTAS=64 timeout 300 python tools/prof_dense.py 3 2 > gpurun_out/prof_c3_64.log 2>&1; echo rc=$?; cat gpurun_out/prof_c3_64.log

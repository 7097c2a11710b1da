timeout 900 python tools/prof_big.py 4 2 > gpurun_out/gate_c4.log 2>&1; echo "C4 rc=$?"; tail -1 gpurun_out/gate_c4.log
timeout 900 python tools/prof_big.py 3 1 > gpurun_out/gate_c3.log 2>&1; echo "C3 rc=$?"; tail -1 gpurun_out/gate_c3.log

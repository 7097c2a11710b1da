# C3/C4 HBM-gate evidence (one chain, whole GPU): 2 C4 systems, 1 C3 system
timeout 400 python tools/prof_big.py 4 2 > gpurun_out/evid_c4.log 2>&1; echo "C4 rc=$?"; tail -1 gpurun_out/evid_c4.log
timeout 400 python tools/prof_big.py 3 1 > gpurun_out/evid_c3.log 2>&1; echo "C3 rc=$?"; tail -1 gpurun_out/evid_c3.log

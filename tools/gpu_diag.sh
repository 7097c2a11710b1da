export SKR_LIB_PATH=$PWD/alt/diag/libskr.so
timeout 900 python tools/c3_chains_probe.py 3 16 8 > gpurun_out/diag_c3.log 2>&1; echo "c3 rc=$?"; grep chunk gpurun_out/diag_c3.log
timeout 600 python tools/c3_chains_probe.py 1 32 8 > gpurun_out/diag_c1.log 2>&1; echo "c1 rc=$?"; grep chunk gpurun_out/diag_c1.log
timeout 600 python tools/c3_chains_probe.py 4 4 2 > gpurun_out/diag_c4.log 2>&1; echo "c4 rc=$?"; grep chunk gpurun_out/diag_c4.log
timeout 600 python tools/c3_chains_probe.py 2 8 4 > gpurun_out/diag_c2.log 2>&1; echo "c2 rc=$?"; grep chunk gpurun_out/diag_c2.log

timeout 300 python tools/prof_big.py 4 1 > gpurun_out/c4_plain.log 2>&1; echo plain_rc=$?; tail -1 gpurun_out/c4_plain.log | cut -c1-300
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_cycle -s 2 -c 1 -o gpurun_out/ncu_c4_cycle python tools/prof_big.py 4 1 > gpurun_out/ncu_c4.log 2>&1; echo ncu_rc=$?; tail -3 gpurun_out/ncu_c4.log

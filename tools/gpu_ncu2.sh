timeout 300 python tools/prof_dense.py 1 1 > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cycle -s 6 -c 1 -o gpurun_out/prof_cycle2 python tools/prof_dense.py 1 1 > gpurun_out/ncu_cycle.log 2>&1; echo ncu1_rc=$?

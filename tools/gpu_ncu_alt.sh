export SKR_LIB_PATH=$PWD/alt/orig/libskr.so
timeout 600 ncu --set full --import-source on --clock-control none --warp-sampling-interval 0 -k regex:^k_dense$ --launch-skip 30 --launch-count 1 -o gpurun_out/kdense_orig -f python tools/prof_dense.py 1 2 > gpurun_out/ncu_kdense.log 2>&1; echo "ncu rc=$?"; tail -1 gpurun_out/ncu_kdense.log

# dense-kernel phase profile + one sampled ncu capture of k_dense (source view)
timeout 300 python tools/prof_dense.py > gpurun_out/prof_dense.log 2>&1; echo "prof_dense rc=$?"; grep -v Warning gpurun_out/prof_dense.log | sed -n 3,20p
timeout 600 ncu --set full --import-source on --clock-control none --warp-sampling-interval 0 -k regex:^k_dense$ --launch-skip 30 --launch-count 1 -o gpurun_out/kdense -f python tools/prof_dense.py 1 2 > gpurun_out/ncu_kdense.log 2>&1; echo "ncu rc=$?"; tail -1 gpurun_out/ncu_kdense.log

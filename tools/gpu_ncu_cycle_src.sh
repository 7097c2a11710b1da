# one k_cycle launch of the bench config with source-level warp sampling
BCMD="bench.py --steps 1 --warmup 3 --stripe 8 --no-cpu-baseline --no-e2e"
timeout 900 ncu --set full --import-source on --clock-control none --warp-sampling-interval 2 -k regex:k_cycle -s 40 -c 1 -o gpurun_out/kcyc_src -f python $BCMD > gpurun_out/ncu_kcyc_src.log 2>&1; echo ncu rc=$?

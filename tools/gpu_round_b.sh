# Evidence pass (part B): one ncu --set full capture of k_cycle in the default bench config.
TAG=${TAG:-r01}
BCMD="bench.py --steps 1 --warmup 3 --stripe 8 --no-cpu-baseline --no-e2e"
timeout 600 python $BCMD > gpurun_out/bench_small_b_$TAG.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_cycle -s 40 -c 1 -o gpurun_out/kcycle_$TAG python $BCMD > gpurun_out/ncu_full_$TAG.log 2>&1; echo ncu_full_rc=$?
tail -3 gpurun_out/ncu_full_$TAG.log

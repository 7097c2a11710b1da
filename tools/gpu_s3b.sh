ALT=regpf CFGS="3 1" bash tools/gpu_ab2.sh
BCMD="bench.py --config 1 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 python $BCMD > gpurun_out/bench_c1_small.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1_s3.csv python $BCMD > gpurun_out/ncu_c1.log 2>&1; echo ncu_rc=$?
python tools/launch_summary.py gpurun_out/launches_c1_s3.csv > gpurun_out/launches_c1_s3_by_kernel.txt; head -12 gpurun_out/launches_c1_s3_by_kernel.txt

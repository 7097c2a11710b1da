# Evidence pass (part A): parity tests, default bench, ncu launch list of a
# short bench (one ncu per call; part B = tools/gpu_round_b.sh).
set -o pipefail
TAG=${TAG:-r01g}
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/pytest_gpu_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.log 2>&1; echo bench_rc=$?
tail -1 gpurun_out/bench_$TAG.log
BCMD="bench.py --steps 1 --warmup 3 --stripe 8 --no-cpu-baseline --no-e2e"
timeout 600 python $BCMD > gpurun_out/bench_small_$TAG.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python $BCMD > gpurun_out/ncu_launch_$TAG.log 2>&1; echo ncu_list_rc=$?
python tools/launch_summary.py gpurun_out/launches_$TAG.csv > gpurun_out/launches_by_kernel_$TAG.txt; head -12 gpurun_out/launches_by_kernel_$TAG.txt

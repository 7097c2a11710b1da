# Evidence pass: parity tests, bench, ncu launch list + one full k_cycle capture.
set -o pipefail
TAG=${TAG:-r01}
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/pytest_gpu_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.log 2>&1; echo bench_rc=$?
tail -1 gpurun_out/bench_$TAG.log
BCMD="bench.py --steps 1 --warmup 1 --stripe 2 --no-cpu-baseline --no-e2e"
timeout 600 python $BCMD > gpurun_out/bench_small_$TAG.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python $BCMD > gpurun_out/ncu_launch_$TAG.log 2>&1; echo ncu_list_rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_cycle -s 20 -c 1 -o gpurun_out/kcycle_$TAG python $BCMD > gpurun_out/ncu_full_$TAG.log 2>&1; echo ncu_full_rc=$?
python tools/launch_summary.py gpurun_out/launches_$TAG.csv | head -12

# Round evidence: parity tests, default bench line, ncu launch list of a short
# bench, ncu --set full of one k_cycle launch (bench config) and one at C4.
set -o pipefail
TAG=${TAG:-r01g}
bash tools/gpu_round.sh
BCMD="bench.py --steps 1 --warmup 3 --stripe 8 --no-cpu-baseline --no-e2e"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_cycle -s 40 -c 1 -o gpurun_out/kcycle_$TAG python $BCMD > gpurun_out/ncu_full_$TAG.log 2>&1; echo ncu_full_rc=$?
timeout 400 python tools/prof_big.py 4 1 > gpurun_out/c4_pre_$TAG.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_cycle -s 3 -c 1 -o gpurun_out/kcycle_c4_$TAG python tools/prof_big.py 4 1 > gpurun_out/ncu_c4_$TAG.log 2>&1; echo ncu_c4_rc=$?

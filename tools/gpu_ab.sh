# A/B of the current build against builds of older revisions (tools/build_alt.sh REV NAME)
# usage: bash tools/gpu_ab.sh NAME [NAME ...]
for v in cur "$@" cur; do
  if [ $v = cur ]; then unset SKR_LIB_PATH; else export SKR_LIB_PATH=$PWD/alt/$v/libskr.so; fi
  timeout 300 python tools/prof_big.py 4 2 > gpurun_out/ab4_$v.log 2>&1; echo "C4 $v rc=$?"; tail -1 gpurun_out/ab4_$v.log | cut -c200-400
  timeout 400 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/abb_$v.log 2>&1; echo "bench $v rc=$?"
  tail -1 gpurun_out/abb_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', round(d['value'],2), 'split', d['time_split_ms'])"
done

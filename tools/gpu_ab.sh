# A/B: current build vs older revisions built by tools/build_alt.sh
for v in cur b66c bd57 cur; do
  if [ $v = cur ]; then unset SKR_LIB_PATH; else export SKR_LIB_PATH=$PWD/alt/$v/libskr.so; fi
  timeout 300 python tools/prof_big.py 4 2 > gpurun_out/ab4_$v.log 2>&1; echo "C4 $v rc=$?"; tail -1 gpurun_out/ab4_$v.log | cut -c200-400
done
for v in cur b66c; do
  if [ $v = cur ]; then unset SKR_LIB_PATH; else export SKR_LIB_PATH=$PWD/alt/$v/libskr.so; fi
  timeout 400 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/abb_$v.log 2>&1; echo "bench $v rc=$?"
  tail -1 gpurun_out/abb_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', round(d['value'],2), 'it', round(d['iterations_mean'],1), 'split', d['time_split_ms'], 'agg', round(d['roofline']['aggregate_gbs']))"
done

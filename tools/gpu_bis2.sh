big() { tag=$1; shift; env "$@" timeout 300 python tools/prof_big.py 4 2 > gpurun_out/bis4_$tag.log 2>&1; echo "C4 $tag rc=$?"; tail -1 gpurun_out/bis4_$tag.log | cut -c230-400; }
big varA SKR_LIB_PATH=$PWD/alt/varA/libskr.so
big cur
big varA2 SKR_LIB_PATH=$PWD/alt/varA/libskr.so
big cur2
timeout 400 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bis_b.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bis_b.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', round(d['value'],2), 'it', round(d['iterations_mean'],1), 'split', d['time_split_ms'], 'agg', round(d['roofline']['aggregate_gbs']))"

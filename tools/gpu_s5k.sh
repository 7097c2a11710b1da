# k_cycle compiled without the fused update (alt/nofuse, k_update direct) vs the default build
run() { timeout 600 python bench.py --config 3 --no-cpu-baseline --no-e2e --gen device 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['value'],3), 'it', round(d['iterations_mean'],2), d['all_converged'], 'launches', d['gpu_launches'])"; }
for rep in 1 2; do
unset SKR_LIB_PATH; run default_fused
export SKR_LIB_PATH=$PWD/alt/nofuse/libskr.so; run nofuse_kupdate; unset SKR_LIB_PATH
done
export SKR_LIB_PATH=$PWD/alt/nofuse/libskr.so
SKR_PROF_CTAS=37 timeout 600 python tools/prof_dense.py 3 2 2>&1 | grep -E "sweep1|sweep2|us/step|START|x update"

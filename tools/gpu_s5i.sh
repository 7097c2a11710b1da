# fused update (default) vs k_update staged vs k_update direct, C3 bench + parity prefix under the new mode
run() { timeout 600 python bench.py --config 3 --no-cpu-baseline --no-e2e --gen device 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', round(d['value'],3), 'it', round(d['iterations_mean'],2), d['all_converged'], 'launches', d['gpu_launches'])"; }
for rep in 1 2; do
unset SKR_FUSE_COMB; unset SKR_UPD_DIRECT; run fused
export SKR_FUSE_COMB=2; export SKR_UPD_DIRECT=0; run kupdate_staged
export SKR_UPD_DIRECT=1; run kupdate_direct
done
export SKR_FUSE_COMB=2; export SKR_UPD_DIRECT=1
timeout 900 python -m pytest tests/test_full_parity.py -k "prefix" -q -s -p no:cacheprovider 2>&1 | grep -E "gpu \[|passed|failed"
timeout 600 python tools/prof_chains.py 3 16 8 37 2>&1 | grep -E "all chains"

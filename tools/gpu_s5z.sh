run() { timeout 600 python bench.py --config $2 --no-cpu-baseline --no-e2e --gen device 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 C$2', round(d['value'],3), 'it', round(d['iterations_mean'],2), d['all_converged'])"; }
for rep in 1 2; do
unset CUDA_DEVICE_MAX_CONNECTIONS; run default 3
export CUDA_DEVICE_MAX_CONNECTIONS=32; run conn32 3; unset CUDA_DEVICE_MAX_CONNECTIONS
done
unset CUDA_DEVICE_MAX_CONNECTIONS; run default 1
export CUDA_DEVICE_MAX_CONNECTIONS=32; run conn32 1

SKR_TRACE=1 timeout 600 python bench.py --config 3 --no-cpu-baseline --no-e2e --gen device > gpurun_out/trace_s5t.log 2>&1
grep "^trace chain 0 sys" gpurun_out/trace_s5t.log | tail -8

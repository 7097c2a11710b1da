export SKR_E2E_DEBUG=1
for i in 1 2 3; do
  timeout 600 python bench.py --no-cpu-baseline > gpurun_out/e2e_dbg_$i.log 2>&1
  grep "e2e phases" gpurun_out/e2e_dbg_$i.log | tail -3
  tail -1 gpurun_out/e2e_dbg_$i.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['e2e']['value'],1))"
done
nproc; cat /sys/fs/cgroup/cpu.max 2>/dev/null

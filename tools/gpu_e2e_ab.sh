for v in 0 1 0 1; do
  if [ $v = 1 ]; then export SKR_E2E_SYNC=1; else unset SKR_E2E_SYNC; fi
  if [ $v = 2 ]; then export SKR_NO_STENCIL=1; else unset SKR_NO_STENCIL; fi
  timeout 600 python bench.py --no-cpu-baseline > gpurun_out/e2e_$v.log 2>&1
  echo -n "sync=$v "; tail -1 gpurun_out/e2e_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['e2e']['value'],1))"
done
export SKR_NO_STENCIL=1; unset SKR_E2E_SYNC
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/e2e_nost.log 2>&1
echo -n "nostencil "; tail -1 gpurun_out/e2e_nost.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['e2e']['value'],1))"

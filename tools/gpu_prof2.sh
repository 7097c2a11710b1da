timeout 600 python tools/prof_dense.py 1 2 > gpurun_out/prof_dense.log 2>&1; echo rc=$?
grep -v "Warn\|return torch" gpurun_out/prof_dense.log
for nb in 64 128 148; do SKR_NBLK=$nb timeout 600 python tools/prof_dense.py 1 2 2>&1 | grep "cycle_ms" | sed "s/^/nblk=$nb /"; done

timeout 600 python tools/prof_dense.py 1 2 > gpurun_out/prof_dense.log 2>&1; echo rc=$?
grep -v "Warn\|return torch" gpurun_out/prof_dense.log
SKR_NBLK=512 timeout 600 python tools/prof_dense.py 1 2 2>&1 | grep "cycle" | sed "s/^/nblk=512 /"

timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/pytest_gpu.log
for nb in 256 296; do echo "== nblk $nb"; SKR_NBLK=$nb timeout 600 python tools/prof_dense.py 1 2 2>&1 | grep -v "Warn\|return torch"; done

# A/B of the dense-kernel phase profile: current build vs alt/<name> builds
for v in cur "$@"; do
  if [ $v = cur ]; then unset SKR_LIB_PATH; else export SKR_LIB_PATH=$PWD/alt/$v/libskr.so; fi
  timeout 300 python tools/prof_dense.py > gpurun_out/abd_$v.log 2>&1; echo "== $v rc=$?"; grep "hqr\|LU\|hessen\|dense_ms" gpurun_out/abd_$v.log
done

# session 4 first pass: full gpu tests, default bench (both arms), C3 launch list
TAG=s4a
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.log 2>&1; echo bench_rc=$?; tail -1 gpurun_out/bench_$TAG.log
timeout 900 python bench.py --gen device > gpurun_out/bench_gendev_$TAG.log 2>&1; echo bench_gendev_rc=$?; tail -1 gpurun_out/bench_gendev_$TAG.log
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_$TAG.log 2>&1; echo ref_rc=$?; tail -1 gpurun_out/bench_ref_$TAG.log
timeout 400 python tools/prof_dense.py 1 3 > gpurun_out/prof_dense_c1.log 2>&1; tail -30 gpurun_out/prof_dense_c1.log
SKR_PROF_CTAS=37 timeout 600 python tools/prof_dense.py 3 2 > gpurun_out/prof_dense_c3.log 2>&1; tail -30 gpurun_out/prof_dense_c3.log

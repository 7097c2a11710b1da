# HEAD (k_gram_dmma build): default bench, both arms, and the full GPU suite once more
timeout 900 python bench.py > gpurun_out/bench_c3_final.log 2>&1; echo bench_rc=$?; tail -1 gpurun_out/bench_c3_final.log | cut -c1-160
timeout 600 python bench.py --impl reference > gpurun_out/bench_c3_ref_final.log 2>&1; echo ref_rc=$?; tail -1 gpurun_out/bench_c3_ref_final.log | cut -c1-160
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_final.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu_final.log

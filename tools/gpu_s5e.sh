# full GPU suite after the preconditioner work + preconditioner timings at C1 / C3 sizes
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_s5e.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_s5e.log
timeout 900 python tools/prof_precond.py 1 3 2>&1 | grep -v Warn | tee gpurun_out/prof_precond_c1.log
timeout 900 python tools/prof_precond.py 3 2 2>&1 | grep -v Warn | tee gpurun_out/prof_precond_c3.log

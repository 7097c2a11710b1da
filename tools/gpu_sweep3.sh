timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
for R in 2 4; do
  export SKR_CYCLE_R=$R
  timeout 300 python tools/prof_big.py 4 2 > gpurun_out/big4_R$R.log 2>&1; echo "C4 R=$R rc=$?"; tail -1 gpurun_out/big4_R$R.log | cut -c1-400
done
unset SKR_CYCLE_R
timeout 400 python tools/prof_big.py 3 1 > gpurun_out/big3.log 2>&1; echo "C3 rc=$?"; tail -1 gpurun_out/big3.log | cut -c1-400
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_cycle -s 2 -c 1 -o gpurun_out/ncu_c4_cycle python tools/prof_big.py 4 1 > gpurun_out/ncu_c4.log 2>&1; echo ncu_rc=$?

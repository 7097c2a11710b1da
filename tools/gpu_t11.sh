timeout 1200 python -m pytest tests/test_full_parity.py -m gpu -q -s -k "c0_full" > gpurun_out/pc0.log 2>&1; echo "c0 rc=$?"; grep -E "C0 chain|passed|failed|Error" gpurun_out/pc0.log | head -5
timeout 600 python tools/c2_gpu_chain.py 545 522 954 830 2>&1 | grep -E "chain|cold"

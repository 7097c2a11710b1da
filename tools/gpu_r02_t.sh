timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python -m pytest tests/test_full_parity.py -m gpu -q -s > gpurun_out/pytest_full.log 2>&1; echo "full rc=$?"; grep -E "gpu \[|passed|failed|Error" gpurun_out/pytest_full.log | head
SKR_FULL_PARITY=1 timeout 1500 python -m pytest tests/test_full_parity.py -m gpu -q -s -k "teacher and 1-16" > gpurun_out/pytest_tf.log 2>&1; echo "tf rc=$?"; grep -E "pos|passed|failed|Error" gpurun_out/pytest_tf.log | head -30

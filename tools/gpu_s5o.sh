# teacher-forced full-size parity with the final build (oracle recomputed on the box) + smoke()
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
SKR_FULL_PARITY=1 timeout 3000 python -m pytest tests/test_full_parity.py -k teacher -q -s -p no:cacheprovider 2>&1 | grep -E "pos|passed|failed" | tee gpurun_out/teacher_forced_final.log

timeout 600 python tools/prof_dense.py 1 3 > gpurun_out/prof_dense.log 2>&1; echo rc=$?
grep -v Warn gpurun_out/prof_dense.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1.csv python tools/prof_dense.py 1 2 > gpurun_out/ncu_plain.log 2>&1; echo ncu_rc=$?
python tools/launch_summary.py gpurun_out/launches_c1.csv

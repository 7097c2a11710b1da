# ncu evidence at the headline config (C3, bench chain shape); reports summarised here, .ncu-rep removed
set -o pipefail
timeout 600 python tools/ncu_capture.py 3 37 > gpurun_out/ncap_plain.log 2>&1; echo "plain rc=$?"; tail -1 gpurun_out/ncap_plain.log
timeout 1800 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none --nvtx --nvtx-include "capture/" -k regex:k_cycle --csv --log-file gpurun_out/kcycle_c3_dram.csv python tools/ncu_capture.py 3 37 > gpurun_out/ncu_dram_c3.log 2>&1; echo "ncu dram rc=$?"; tail -1 gpurun_out/ncu_dram_c3.log
timeout 1800 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "capture/" -k regex:k_cycle -s 5 -c 1 -o /tmp/kcycle_c3_full python tools/ncu_capture.py 3 37 > gpurun_out/ncu_full_c3.log 2>&1; echo "ncu full rc=$?"
python tools/ncu_summary.py /tmp/kcycle_c3_full.ncu-rep gpurun_out/ncu_k_cycle_c3_full > /dev/null 2>&1; echo "summary rc=$?"
ncu -i /tmp/kcycle_c3_full.ncu-rep --page details > gpurun_out/ncu_k_cycle_c3_details.txt 2>&1
ncu -i /tmp/kcycle_c3_full.ncu-rep --page source --csv > /tmp/src.csv 2>&1; python tools/ncu_lines.py /tmp/src.csv > gpurun_out/ncu_k_cycle_c3_lines.txt 2>&1; echo "lines rc=$?"
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu launch rc=$?"
python tools/launch_summary.py /tmp/launches.csv > gpurun_out/launches_c3_r02_by_kernel.txt; head -8 gpurun_out/launches_c3_r02_by_kernel.txt
gzip -c /tmp/launches.csv > gpurun_out/launches_c3_r02.csv.gz
du -sh gpurun_out

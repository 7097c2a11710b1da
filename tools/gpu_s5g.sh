# alone (1 chain x 37 CTAs) phase profile incl. the cycle-start points; ncu source-level capture of one deflated k_cycle
SKR_PROF_CTAS=37 timeout 600 python tools/prof_dense.py 3 2 2>&1 | grep -v Warn | tail -16
timeout 1800 ncu --set full --clock-control none --import-source on --warp-sampling-interval 3 --nvtx --nvtx-include "capture/" -k regex:k_cycle -s 5 -c 1 -f -o /tmp/kcyc_src python tools/ncu_capture.py 3 37 > gpurun_out/ncu_src_s5g.log 2>&1; echo "ncu rc=$?"
ncu -i /tmp/kcyc_src.ncu-rep --page source --csv --print-source=sass > gpurun_out/kcyc_src_sass.csv 2>&1; echo "csv rc=$?"; ls -la gpurun_out/kcyc_src_sass.csv
ncu -i /tmp/kcyc_src.ncu-rep --page details 2>&1 | grep -E "Duration|DRAM Throughput|Registers Per|Achieved Occupancy|Executed Ipc|Issue Slots Busy|L1/TEX Hit|L2 Hit|Mem Busy|Max Bandwidth" | head -20

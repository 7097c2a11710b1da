# round-2 final evidence: GPU tests, bench arms, per-config bench lines, ncu captures (C3 bench shape)
TAG=final
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_c3_$TAG.log 2>&1; echo bench_rc=$?; tail -1 gpurun_out/bench_c3_$TAG.log | cut -c1-400
timeout 900 python bench.py --gen device > gpurun_out/bench_c3_gendev_$TAG.log 2>&1; echo bench_gendev_rc=$?; tail -1 gpurun_out/bench_c3_gendev_$TAG.log | cut -c1-200
timeout 600 python bench.py --impl reference > gpurun_out/bench_c3_ref_$TAG.log 2>&1; echo ref_rc=$?; tail -1 gpurun_out/bench_c3_ref_$TAG.log | cut -c1-200
for c in 1 4 0 2; do
timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_c${c}_$TAG.log 2>&1; echo "bench c$c rc=$?"; tail -1 gpurun_out/bench_c${c}_$TAG.log | cut -c1-200
done
# ncu (each after the plain run exited 0)
timeout 600 python tools/ncu_capture.py 3 37 > gpurun_out/ncap_plain.log 2>&1; echo "plain rc=$?"; tail -1 gpurun_out/ncap_plain.log
timeout 1800 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none --nvtx --nvtx-include "capture/" -k regex:k_cycle --csv --log-file gpurun_out/kcycle_c3_dram.csv python tools/ncu_capture.py 3 37 > gpurun_out/ncu_dram_c3.log 2>&1; echo "ncu dram rc=$?"; tail -1 gpurun_out/ncu_dram_c3.log
timeout 1800 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "capture/" -k regex:k_cycle -s 5 -c 1 -f -o /tmp/kcycle_c3_full python tools/ncu_capture.py 3 37 > gpurun_out/ncu_full_c3.log 2>&1; echo "ncu full rc=$?"
python tools/ncu_summary.py /tmp/kcycle_c3_full.ncu-rep gpurun_out/ncu_k_cycle_c3_full > /dev/null 2>&1; echo "summary rc=$?"
ncu -i /tmp/kcycle_c3_full.ncu-rep --page details > gpurun_out/ncu_k_cycle_c3_details.txt 2>&1
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu launch rc=$?"
python tools/launch_summary.py /tmp/launches.csv > gpurun_out/launches_c3_r02_by_kernel.txt; head -8 gpurun_out/launches_c3_r02_by_kernel.txt
gzip -c /tmp/launches.csv > gpurun_out/launches_c3_r02.csv.gz
cuobjdump -sass paper_2401_09516_b200/libskr.so 2>/dev/null | grep -c "DMMA" 
du -sh gpurun_out

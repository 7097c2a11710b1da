CS=/usr/local/cuda/bin/compute-sanitizer
python tools/sanitize_probe.py > gpurun_out/san_plain.log 2>&1; echo "plain rc=$?"; tail -2 gpurun_out/san_plain.log
for tool in memcheck racecheck synccheck; do
  timeout 1500 $CS --tool $tool --print-limit 50 python tools/sanitize_probe.py > gpurun_out/san_$tool.log 2>&1; echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|hazard|Invalid|Error" gpurun_out/san_$tool.log | sort | uniq -c | head -8
done

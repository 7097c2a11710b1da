# ncu --set full of the new kernels: k_gram_dmma (refresh, C3 37 CTAs), k_pc_apply and k_pc_build (C3 ILU(0)), k_update
timeout 900 ncu --set full --clock-control none --nvtx --nvtx-include "capture/" -k regex:k_gram_dmma -c 1 -f -o /tmp/kgram python tools/ncu_capture.py 3 37 > gpurun_out/ncu_kgram.log 2>&1; echo "kgram rc=$?"
python tools/ncu_summary.py /tmp/kgram.ncu-rep gpurun_out/ncu_k_gram_dmma_c3 > /dev/null 2>&1; cat gpurun_out/ncu_k_gram_dmma_c3.md | tail -2
timeout 900 ncu --set full --clock-control none -k regex:k_pc_apply -s 2 -c 1 -f -o /tmp/kpc python tools/prof_pc_apply.py 3 > gpurun_out/ncu_kpc.log 2>&1; echo "kpc rc=$?"
python tools/ncu_summary.py /tmp/kpc.ncu-rep gpurun_out/ncu_k_pc_apply_c3 > /dev/null 2>&1; cat gpurun_out/ncu_k_pc_apply_c3.md | tail -2
timeout 900 ncu --set full --clock-control none -k regex:k_pc_build -c 2 -f -o /tmp/kpcb python tools/prof_pc_apply.py 3 > gpurun_out/ncu_kpcb.log 2>&1; echo "kpcb rc=$?"
python tools/ncu_summary.py /tmp/kpcb.ncu-rep gpurun_out/ncu_k_pc_build_c3 > /dev/null 2>&1; cat gpurun_out/ncu_k_pc_build_c3.md | tail -3
SKR_FUSE_COMB=2 timeout 900 ncu --set full --clock-control none --nvtx --nvtx-include "capture/" -k regex:k_update -s 3 -c 1 -f -o /tmp/kupd python tools/ncu_capture.py 3 37 > gpurun_out/ncu_kupd.log 2>&1; echo "kupd rc=$?"
python tools/ncu_summary.py /tmp/kupd.ncu-rep gpurun_out/ncu_k_update_c3 > /dev/null 2>&1; cat gpurun_out/ncu_k_update_c3.md | tail -2

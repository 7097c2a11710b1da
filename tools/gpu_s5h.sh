# A/B: vectorised apply_update staging (cur) vs HEAD (alt/prev): C3 bench, alone profile
ALT=prev CFGS="3" bash tools/gpu_ab2.sh
SKR_PROF_CTAS=37 timeout 600 python tools/prof_dense.py 3 2 2>&1 | grep -E "sweep1|sweep2|us/step|START|x update"

# sweep 2 as a noinline function with 16-column batches (cur) vs HEAD (alt/prev)
ALT=prev CFGS="3" bash tools/gpu_ab2.sh
SKR_PROF_CTAS=37 timeout 600 python tools/prof_dense.py 3 2 2>&1 | grep -E "sweep1|sweep2|us/step|START|x update"

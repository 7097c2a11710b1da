big() { tag=$1; shift; env "$@" timeout 300 python tools/prof_big.py 4 2 > gpurun_out/pad4_$tag.log 2>&1; echo "C4 $tag rc=$?"; tail -1 gpurun_out/pad4_$tag.log | cut -c230-400; }
big p0
big p40k SKR_SMEM_PAD=40960
big p20k SKR_SMEM_PAD=20480
big p60k SKR_SMEM_PAD=61440
big p40k_co100 SKR_SMEM_PAD=40960 SKR_CARVEOUT=100
big b66c SKR_LIB_PATH=$PWD/alt/b66c/libskr.so

big() { tag=$1; shift; env "$@" timeout 300 python tools/prof_big.py 4 2 > gpurun_out/bis4_$tag.log 2>&1; echo "C4 $tag rc=$?"; tail -1 gpurun_out/bis4_$tag.log | cut -c230-400; }
big b66c SKR_LIB_PATH=$PWD/alt/b66c/libskr.so
big varA SKR_LIB_PATH=$PWD/alt/varA/libskr.so
big varB SKR_LIB_PATH=$PWD/alt/varB/libskr.so
big cur
big b66c2 SKR_LIB_PATH=$PWD/alt/b66c/libskr.so

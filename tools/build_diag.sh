# build the working tree's libskr.so with extra flags into alt/$1/libskr.so
# usage: bash tools/build_diag.sh NAME "-DSKR_DIAG ..."
set -e
NAME=$1; FLAGS=$2
D=/tmp/skr_diag_$NAME; rm -rf $D; mkdir -p $D
mkdir -p /root/repo/alt/$NAME
C=/root/repo/paper_2401_09516_b200/csrc
for f in gcrodr sort assemble; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC $FLAGS -I /root/repo/include -c $C/$f.cu -o $D/$f.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o /root/repo/alt/$NAME/libskr.so $D/gcrodr.o $D/sort.o $D/assemble.o -lcudart_static -lrt -ldl -lpthread
echo built /root/repo/alt/$NAME/libskr.so

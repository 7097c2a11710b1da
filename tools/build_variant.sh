# build the working tree's libskr.so with extra nvcc flags into alt/$1/libskr.so
set -e
NAME=$1; shift
D=/root/repo/alt/$NAME; mkdir -p $D
cd /root/repo/paper_2401_09516_b200/csrc
for f in gcrodr sort assemble; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I /root/repo/include "$@" -c $f.cu -o $D/$f.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $D/libskr.so $D/gcrodr.o $D/sort.o $D/assemble.o -lcudart_static -lrt -ldl -lpthread
rm -f $D/*.o
echo built $D/libskr.so

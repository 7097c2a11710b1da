# build libskr.so of git revision $1 into alt/$2/libskr.so (A/B measurements)
set -e
REV=$1; NAME=$2
D=/tmp/skr_alt_$NAME; rm -rf $D; mkdir -p $D
git -C /root/repo archive $REV paper_2401_09516_b200/csrc include | tar -x -C $D
mkdir -p /root/repo/alt/$NAME
cd $D/paper_2401_09516_b200/csrc
FILES=$(cd $D/paper_2401_09516_b200/csrc && ls *.cu | sed 's/\.cu$//')
for f in $FILES; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I $D/include -c $f.cu -o $D/$f.o
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o /root/repo/alt/$NAME/libskr.so $(for f in $FILES; do echo $D/$f.o; done) -lcudart_static -lrt -ldl -lpthread
echo built /root/repo/alt/$NAME/libskr.so

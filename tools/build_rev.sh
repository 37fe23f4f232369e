# usage: bash tools/build_rev.sh <git-rev> <out.so>   (the product library at another revision; A/B via SYMM_LIB=<out.so>)
set -e
rev=$1; out=$2
d=$(mktemp -d); mkdir -p $d/include $d/csrc
git show $rev:include/symmspmv.h > $d/include/symmspmv.h
for f in schedule.cpp cs_build.cpp capi.cpp kernels.cu internal.h; do git show $rev:paper_1907_06487_b200/csrc/$f > $d/csrc/$f; done
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-fopenmp,-O3 --expt-relaxed-constexpr -I$d/include -I$d/csrc"
g++ -O3 -std=c++17 -fopenmp -fPIC -I$d/include -I$d/csrc -c -o $d/schedule.o $d/csrc/schedule.cpp
g++ -O3 -std=c++17 -fopenmp -fPIC -I$d/include -I$d/csrc -c -o $d/cs_build.o $d/csrc/cs_build.cpp
nvcc $F -x cu -c -o $d/capi.o $d/csrc/capi.cpp
nvcc $F -c -o $d/kernels.o $d/csrc/kernels.cu
mkdir -p $(dirname $out)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fopenmp -o $out $d/schedule.o $d/cs_build.o $d/capi.o $d/kernels.o -lcudart
rm -rf $d

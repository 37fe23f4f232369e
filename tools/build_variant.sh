# usage: bash tools/build_variant.sh <out.so> <kernels.cu> [internal.h] [capi.cpp]
# builds the product library with alternative sources (A/B diagnostics; SYMM_LIB=<out.so>)
set -e
out=$1; kc=$2; ih=${3:-paper_1907_06487_b200/csrc/internal.h}; cc=${4:-paper_1907_06487_b200/csrc/capi.cpp}
d=$(mktemp -d); cp paper_1907_06487_b200/csrc/*.cpp paper_1907_06487_b200/csrc/*.h $d/; cp $kc $d/kernels.cu; cp $ih $d/internal.h; cp $cc $d/capi.cpp
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-fopenmp,-O3 --expt-relaxed-constexpr -Iinclude -I$d"
g++ -O3 -std=c++17 -fopenmp -fPIC -Iinclude -I$d -c -o $d/schedule.o $d/schedule.cpp
g++ -O3 -std=c++17 -fopenmp -fPIC -Iinclude -I$d -c -o $d/cs_build.o $d/cs_build.cpp
nvcc $F -x cu -c -o $d/capi.o $d/capi.cpp
nvcc $F -c -o $d/kernels.o $d/kernels.cu
mkdir -p $(dirname $out)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fopenmp -o $out $d/schedule.o $d/cs_build.o $d/capi.o $d/kernels.o -lcudart
rm -rf $d

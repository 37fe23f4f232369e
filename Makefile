# Builds the three native libraries in-tree (they travel to the GPU box with
# the gpurun snapshot; *.so is git-ignored):
#   gen/libsymmgen.so                      seeded input generators (shared by tests + bench)
#   oracle/liboracle.so                    CPU oracle (tests / smoke / cpu_baseline only)
#   paper_1907_06487_b200/libsymmspmv.so   the product: C-ABI schedule builder + sm_100a kernels
NVCC ?= nvcc
CXX ?= g++
CC ?= gcc
# host C++ compiler with OpenMP: the first of $(CXX), g++, /usr/bin/g++ that
# links -fopenmp (some images point CXX at a wrapper without libgomp.spec)
OMPCXX := $(shell for c in $(CXX) g++ /usr/bin/g++; do echo 'int main(){return 0;}' | $$c -fopenmp -x c++ - -o /dev/null >/dev/null 2>&1 && { echo $$c; break; }; done)
OMPCC := $(shell for c in $(CC) gcc /usr/bin/gcc; do echo 'int main(){return 0;}' | $$c -fopenmp -x c - -o /dev/null >/dev/null 2>&1 && { echo $$c; break; }; done)
ifeq ($(OMPCXX),)
$(error no host C++ compiler with OpenMP support found)
endif
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) $(EXTRA_NVFLAGS) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-fopenmp,-O3 -Xptxas -v --expt-relaxed-constexpr
PKG := paper_1907_06487_b200
CSRC := $(PKG)/csrc

PROD_SRCS := $(CSRC)/schedule.cpp $(CSRC)/cs_build.cpp $(CSRC)/capi.cpp $(CSRC)/kernels.cu
PROD_HDRS := include/symmspmv.h $(CSRC)/internal.h

all: gen/libsymmgen.so oracle/liboracle.so $(PKG)/libsymmspmv.so

gen/libsymmgen.so: gen/symmgen.cpp
	$(OMPCXX) -O2 -std=c++17 -fopenmp -fPIC -shared -Wall -o $@ $<

# -ffp-contract=off: no FMA contraction in the oracle (reading R5)
oracle/liboracle.so: oracle/oracle.c
	$(OMPCC) -O2 -std=c99 -ffp-contract=off -fopenmp -fPIC -shared -Wall -o $@ $<

$(CSRC)/schedule.o: $(CSRC)/schedule.cpp $(PROD_HDRS)
	$(OMPCXX) -O3 -std=c++17 -fopenmp -fPIC -Wall -Iinclude -c -o $@ $<

$(CSRC)/cs_build.o: $(CSRC)/cs_build.cpp $(PROD_HDRS)
	$(OMPCXX) -O3 -std=c++17 -fopenmp -fPIC -Wall -Iinclude -c -o $@ $<

$(CSRC)/capi.o: $(CSRC)/capi.cpp $(PROD_HDRS)
	$(NVCC) $(NVFLAGS) -Iinclude -x cu -c -o $@ $<

$(CSRC)/kernels.o: $(CSRC)/kernels.cu $(PROD_HDRS)
	$(NVCC) $(NVFLAGS) -Iinclude -c -o $@ $< 2> $(CSRC)/ptxas.log || (cat $(CSRC)/ptxas.log; false)

$(PKG)/libsymmspmv.so: $(CSRC)/schedule.o $(CSRC)/cs_build.o $(CSRC)/capi.o $(CSRC)/kernels.o
	$(NVCC) $(ARCH) -shared -Xcompiler -fopenmp -o $@ $^ -lcudart

clean:
	rm -f gen/*.so oracle/*.so $(PKG)/*.so $(CSRC)/*.o

.PHONY: all clean

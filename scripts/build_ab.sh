#!/bin/bash
# A/B library: the W=1 search kernels rebuilt with extra -D flags, linked with the rest of the
# in-tree objects into _ab/libcubics.so (load it with CUBICS_LIB=$PWD/_ab/libcubics.so)
set -e
cd "$(dirname "$0")/../paper_1909_09213_b200/csrc"
mkdir -p ../../_ab/obj
/usr/local/cuda/bin/nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC,-O3 \
  -ccbin /usr/bin/g++ -I../../include -DCUBICS_W=1 -DCUBICS_PART=0 "$@" -Xptxas -v -c kernels_inst.cu \
  -o ../../_ab/obj/kernels_w1_p0.o 2> ../../_ab/obj/ptxas.log
objs=$(ls ../lib/obj/*.o | grep -v kernels_w1_p0.o)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -ccbin /usr/bin/g++ -o ../../_ab/libcubics.so \
  $objs ../../_ab/obj/kernels_w1_p0.o -lcudart -lpthread
echo built _ab/libcubics.so

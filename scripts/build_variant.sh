#!/bin/bash
# Experiment build: the library with gemm_sm100.cu compiled under extra defines.
# usage: [SRC=alt_gemm.cu] scripts/build_variant.sh OUT.so -DFOO=1 ...   (objects of the other sources reused)
set -e
out=$1; shift
B=paper_2402_19481_b200
mkdir -p ab
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC,-fvisibility=hidden \
  -I$B/csrc -Iinclude -DPP_BUILDING_LIB "$@" -c ${SRC:-$B/csrc/gemm_sm100.cu} -o ab/gemm_variant.o
objs=$(ls $B/build/*.o | grep -v gemm_sm100)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out $objs ab/gemm_variant.o -lcudart -lnccl -ldl -lpthread

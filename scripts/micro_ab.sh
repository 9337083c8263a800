#!/bin/bash
# gemm_micro.py under several builds of the library (LIBS), twice each, alternating.
mkdir -p gpurun_out
for rep in 1 2; do
  for lib in ${LIBS:-paper_2402_19481_b200/libpp_b200.so}; do
    echo "== $lib rep $rep"
    PP_B200_LIB=$lib timeout 300 python scripts/gemm_micro.py 2>&1 | head -6
  done
done 2>&1 | tee gpurun_out/micro_ab.txt

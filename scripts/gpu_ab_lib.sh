#!/bin/bash
mkdir -p gpurun_out
{ TAG=old PP_B200_LIB=$PWD/scratch_old/libpp_b200.so timeout 300 python scripts/gemm_ab.py
  TAG=new timeout 300 python scripts/gemm_ab.py
  TAG=k1 PP_KPS=1 timeout 300 python scripts/gemm_ab.py
  TAG=nopdl PP_PDL=0 timeout 300 python scripts/gemm_ab.py; } 2>&1 | tee gpurun_out/ab_lib.txt

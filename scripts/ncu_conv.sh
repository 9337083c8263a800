#!/bin/bash
# Full ncu capture of the first conv GEMM launches of one 1-step generation (1 GPU).
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s ${SKIP:-1} -c ${COUNT:-3} \
  -o gpurun_out/prof_conv -f python bench.py --steps 1 --warmup 0 --num-steps 2 --no-cpu-baseline > gpurun_out/ncu_conv.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/ncu_conv.log

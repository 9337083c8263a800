#!/bin/bash
# Conv-kernel probe on the GPU box: per-launch breakdown of one 1024^2 UNet step (CUPTI),
# the layer-shape micro-benchmark, and one ncu --set full capture of the L01 conv with the
# SASS source page (warp-stall samples per instruction: where the MMA / TMA warps wait).
set -u
mkdir -p gpurun_out
R=${R:-r02e}
{
timeout 300 python scripts/step_breakdown.py 128 bf16 1 0 > gpurun_out/${R}_step_128.txt 2>&1
echo "step breakdown rc=$?"; head -60 gpurun_out/${R}_step_128.txt
timeout 300 python scripts/gemm_micro.py > gpurun_out/${R}_micro.txt 2>&1
echo "micro rc=$?"; cat gpurun_out/${R}_micro.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 3 -c 1 \
  -o gpurun_out/${R}_conv_l01 -f python scripts/gemm_one.py 1 128 128 320 320 0 0 1048578 \
  > gpurun_out/${R}_conv_l01.log 2>&1
echo "ncu rc=$?"
ncu -i gpurun_out/${R}_conv_l01.ncu-rep --page details > gpurun_out/${R}_conv_l01.details.txt 2>/dev/null
ncu -i gpurun_out/${R}_conv_l01.ncu-rep --page raw --csv > gpurun_out/${R}_conv_l01.raw.csv 2>/dev/null
ncu -i gpurun_out/${R}_conv_l01.ncu-rep --page source --csv --print-source sass \
  > gpurun_out/${R}_conv_l01.sass.csv 2>/dev/null
echo "export rc=$?"
} 2>&1 | tee gpurun_out/${R}_probe.txt

#!/bin/bash
# ncu launch lists (gpu__time_duration per launch, serialised, cold cache) of one generation at
# each latent given, e.g.  R=r02a LATENTS="128 480" bash scripts/launch_lists.sh
mkdir -p gpurun_out
for L in ${LATENTS:-128}; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
    --log-file gpurun_out/${R}_launches_$L.csv python scripts/one_generation.py $L ${DTYPE:-bf16} \
    > gpurun_out/${R}_launches_$L.log 2>&1
  echo "launch list $L rc=$?"
  python scripts/launch_summary.py gpurun_out/${R}_launches_$L.csv > gpurun_out/${R}_launches_${L}_summary.txt
  head -20 gpurun_out/${R}_launches_${L}_summary.txt
done

#!/bin/bash
# Full ncu capture of kernels matching $KREGEX (skip $SKIP, count $COUNT) in a 2-step generation.
mkdir -p gpurun_out
OUT=${OUT:-prof_k}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KREGEX} -s ${SKIP:-0} -c ${COUNT:-2} \
  -o gpurun_out/${OUT} -f python bench.py --steps 1 --warmup 0 --num-steps 2 --no-cpu-baseline > gpurun_out/${OUT}.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/${OUT}.log

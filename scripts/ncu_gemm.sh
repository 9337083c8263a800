#!/bin/bash
# ncu --set full of single gemm_kernel launches (args: name kind m w k n force bn reps) from $CASES
mkdir -p gpurun_out
run() {  # name args...
  local name=$1; shift
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 3 -c 1 \
    -o gpurun_out/$name -f python scripts/gemm_one.py "$@" > gpurun_out/$name.log 2>&1
  echo "$name rc=$?"
  ncu -i gpurun_out/$name.ncu-rep --page raw --csv > gpurun_out/$name.raw.csv 2>/dev/null
  ncu -i gpurun_out/$name.ncu-rep --page source --csv --print-source sass > gpurun_out/$name.sass.csv 2>/dev/null
}
run g_l11_gn 1 64 64 640 640 0 0 1048578
run g_l11_nogn 1 64 64 640 640 0 0 2

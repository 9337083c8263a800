#!/bin/bash
# Round measurement on the GPU box: GPU suite, smoke, full bench line, ncu launch list of one
# generation, ncu --set full of the dominant conv kernel (L37 / L01 shapes) and the GN pass.
set -u
mkdir -p gpurun_out
R=${ROUND:-r01c}
{
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 900 python bench.py 2> gpurun_out/bench_$R.err | tail -1 > gpurun_out/bench_$R.json
cat gpurun_out/bench_$R.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1800 --csv \
  --log-file gpurun_out/launches_$R.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline \
  > gpurun_out/ncu_list_$R.log 2>&1; echo "ncu list rc=$?"
for spec in "conv_l37 1 64 64 1280 640 0 0 1048578" "conv_l01 1 128 128 320 320 0 0 1048578"; do
  set -- $spec; name=$1; shift
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 3 -c 1 \
    -o gpurun_out/${R}_$name -f python scripts/gemm_one.py "$@" > gpurun_out/${R}_$name.log 2>&1
  ncu -i gpurun_out/${R}_$name.ncu-rep --page raw --csv > gpurun_out/${R}_$name.raw.csv 2>/dev/null
  ncu -i gpurun_out/${R}_$name.ncu-rep --page details > gpurun_out/${R}_$name.details.txt 2>/dev/null
  echo "ncu $name rc=$?"
done
timeout 300 ncu --set full --clock-control none -k regex:gn_pass -s 5 -c 1 -o gpurun_out/${R}_gn -f \
  python scripts/gn_one.py 16384 320 7 > gpurun_out/${R}_gn.log 2>&1
ncu -i gpurun_out/${R}_gn.ncu-rep --page details > gpurun_out/${R}_gn.details.txt 2>/dev/null
ncu -i gpurun_out/${R}_gn.ncu-rep --page raw --csv > gpurun_out/${R}_gn.raw.csv 2>/dev/null
} 2>&1 | tee gpurun_out/round_$R.txt

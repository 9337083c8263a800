#!/bin/bash
# Round-2 measurement on the GPU box: full bench line, ncu launch list of one 128^2 generation,
# ncu --set full captures of the dominant conv (L01 shape), the attention kernels (S GEMM with
# the softmax epilogue, attn_rescale, PV GEMM with V MN-major) at 128^2 and 480^2, the
# GroupNorm pass and the stem im2col.
set -u
mkdir -p gpurun_out
R=${ROUND:-r02d}
{
if [ -z "${ONLY_CAPS:-}" ]; then
timeout 1200 python bench.py 2> gpurun_out/bench_$R.err | tail -1 > gpurun_out/bench_$R.json
echo "bench rc=$?"; tail -c 300 gpurun_out/bench_$R.json; echo
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
  --log-file gpurun_out/${R}_launches_128.csv python scripts/one_generation.py 128 > gpurun_out/${R}_launches.log 2>&1
echo "launch list rc=$?"
python scripts/launch_summary.py gpurun_out/${R}_launches_128.csv > gpurun_out/${R}_launches_128_summary.txt
head -16 gpurun_out/${R}_launches_128_summary.txt
fi
cap() {   # name, ncu filter args..., -- command
  local name=$1; shift
  timeout 600 ncu --set full --clock-control none --import-source on -o gpurun_out/${R}_$name -f "$@" \
    > gpurun_out/${R}_$name.log 2>&1
  echo "ncu $name rc=$?"
  ncu -i gpurun_out/${R}_$name.ncu-rep --page details > gpurun_out/${R}_$name.details.txt 2>/dev/null
  ncu -i gpurun_out/${R}_$name.ncu-rep --page raw --csv > gpurun_out/${R}_$name.raw.csv 2>/dev/null
}
[ -z "${ONLY_CAPS:-}" ] && cap conv_l01 -k regex:gemm_kernel -s 3 -c 1 python scripts/gemm_one.py 1 128 128 320 320 0 0 1048578
cap attn128 -k regex:"gemm_kernel|attn_rescale" -s 9 -c 3 python scripts/one_generation.py 128
cap attn480 -k regex:"gemm_kernel|attn_rescale" -s 9 -c 3 python scripts/one_generation.py 480
[ -z "${ONLY_CAPS:-}" ] && cap gn -k regex:gn_pass -s 5 -c 1 python scripts/gn_one.py 16384 320 7
cap stem -k regex:"stem_im2col|gemm_kernel" -c 2 python scripts/one_generation.py 128
} 2>&1 | tee gpurun_out/round_$R.txt

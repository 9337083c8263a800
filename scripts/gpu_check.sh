#!/bin/bash
# GPU-box helper: parity tests, one bench line, and the ncu launch list of one generation.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -15
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -4
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 3000 gpurun_out/bench.json; tail -5 gpurun_out/bench.err
if [ "${NCU:-0}" = "1" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4200 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline \
    > gpurun_out/ncu_bench.log 2>&1; echo "ncu rc=$?"; wc -l gpurun_out/launches.csv
fi

#!/bin/bash
# A/B of bench.py under environment variants, e.g.
#   VARIANTS="PP_PDL=0 PP_PDL=1"   (each variant: space-free env assignments joined by ',')
mkdir -p gpurun_out
for v in ${VARIANTS:-"PP_PDL=0" "PP_PDL=1"}; do
  for rep in 1 2; do
    env ${v//,/ } timeout 180 python bench.py --steps 5 --warmup 3 --no-cpu-baseline ${BENCH_ARGS:-} 2>/dev/null | tail -1 > gpurun_out/ab.json
    python -c "
import json; d=json.load(open('gpurun_out/ab.json')); print('$v', 'rep $rep', round(d['value']*1e3,3), 'ms  e2e', round(d['e2e']['value']*1e3,3), 'clk', d['clocks']['sm_mhz'])"
  done
done 2>&1 | tee gpurun_out/ab.txt

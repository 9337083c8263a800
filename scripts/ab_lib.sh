#!/bin/bash
# A/B of two builds of the library on one box: LIBS="ab/libpp_head.so paper_2402_19481_b200/libpp_b200.so"
# alternating runs of bench.py (--no-extras), ms per generation and e2e.
mkdir -p gpurun_out
for rep in 1 2 3; do
  for lib in ${LIBS:-ab/libpp_head.so paper_2402_19481_b200/libpp_b200.so}; do
    PP_B200_LIB=$lib timeout 300 python bench.py --steps ${STEPS:-8} --warmup 3 --no-cpu-baseline --no-extras ${BENCH_ARGS:-} 2>/dev/null | tail -1 > gpurun_out/ab.json
    python -c "
import json; d=json.load(open('gpurun_out/ab.json')); print('$lib', 'rep $rep', round(d['value']*1e3,3), 'ms  e2e', round(d['e2e']['value']*1e3,3), 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'])"
  done
done 2>&1 | tee gpurun_out/ab_lib.txt

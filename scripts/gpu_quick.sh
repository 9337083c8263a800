#!/bin/bash
# GPU-box helper: GEMM parity + micro-benchmarks, then selected runner tests (each under a timeout).
set -u
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gemm_gpu.py -q -x 2>&1 | tail -5
timeout 300 python scripts/gemm_micro.py ${MICRO_ARGS:-} 2>&1 | tail -20
timeout 600 python -X faulthandler -m pytest tests/test_runner_gpu.py -q -x ${RUNNER_ARGS:-} > gpurun_out/runner.log 2>&1; echo "runner rc=$?"
grep -m3 -B2 -A30 "Fatal Python error\|Error\|FAILED" gpurun_out/runner.log | head -80
tail -3 gpurun_out/runner.log

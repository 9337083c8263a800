#!/bin/bash
# GPU-box helper: GEMM/conv kernel parity (single CTA + CTA pair), micro-benchmarks.
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gemm_gpu.py -q -x 2>&1 | tail -8
timeout 600 python scripts/gemm_micro.py ${MICRO_ARGS:---cta} 2>&1 | tail -80

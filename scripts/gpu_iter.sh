#!/bin/bash
# GPU-box iteration helper: GEMM parity + micro-benchmarks (+ an env variant), full GPU suite,
# one bench line.  Everything also lands in gpurun_out/iter.txt.
set -u
mkdir -p gpurun_out
{
timeout 600 python -m pytest tests/test_gemm_gpu.py -q -x 2>&1 | tail -4
timeout 300 python scripts/gemm_micro.py ${MICRO_ARGS:-} 2>&1
if [ -n "${ALT:-}" ]; then echo "--- $ALT"; env $ALT timeout 300 python scripts/gemm_micro.py 2>&1 | head -9; fi
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>gpurun_out/bench.err | tail -1 > gpurun_out/bench.json
python - <<'PY'
import json
d=json.load(open("gpurun_out/bench.json"))
r=d["roofline"]
print("BENCH value", d["value"], "e2e", d["e2e"]["value"], "conv TF/s", r["achieved"], "frac", r["frac"],
      "conv_ms", r.get("conv_ms_per_generation"), "gn_ms", r.get("gn_ms_per_generation"), "clocks", d["clocks"])
PY
} 2>&1 | tee gpurun_out/iter.txt

"""One SDXL-shape generation through the runner (for ncu launch lists / captures).

usage: python scripts/one_generation.py [LATENT] [DTYPE] [BANDS]
The first sample() captures the denoising loop into a CUDA graph and replays it once: the
kernels of exactly one 50-step generation run (plus the per-runner prologue kernels).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2402_19481_b200 import patchsim as P  # noqa: E402

hw = int(sys.argv[1]) if len(sys.argv) > 1 else 128
dtype = sys.argv[2] if len(sys.argv) > 2 else "bf16"
bands = int(sys.argv[3]) if len(sys.argv) > 3 else 1
m = P.build_model(P.SDXL_SHAPE, 42)
cond = P.random_condition(2048, 7)
r = P.PatchRunner(m, cond, hw, hw, mode="displaced", n_devices=bands, warmup_steps=4, dtype=dtype)
x0, _ = r.sample(P.random_normal(1, 4, hw, hw, 1234), P.make_plan(1000, 50), P.make_schedule(1000))
print("ok", float(abs(x0).mean()), r.last_device_ms(), "ms")

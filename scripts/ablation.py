"""Ablation (BASELINE.json configs[4]): naive patch vs synchronous patch parallel vs displaced
(stale, warm-up 4) at 1024^2 (128^2 latent), SDXL-shape, 50-step DDIM, N bands — on ONE B200
(bands run in-process, so times are not multi-GPU scaling numbers).  Reports x0 fidelity vs the
single-device reference run (rel-L2, PSNR over the reference's range) and device ms."""
import json
import math
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2402_19481_b200 import artifacts as A  # noqa: E402
from paper_2402_19481_b200 import patchsim as P  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8
H = W = int(sys.argv[2]) if len(sys.argv) > 2 else 128
cfg = P.SDXL_SHAPE
model = P.build_model(cfg, 42)
cond = P.random_condition(2048, 7)
x_T = P.random_normal(1, 4, H, W, 1234)
abar = P.make_schedule(1000)
plan = P.make_plan(1000, 50)
out = {}
for mode, nd in (("reference", 1), ("sync-pp", n), ("displaced", n), ("naive", n)):
    r = P.PatchRunner(model, cond, H, W, mode=mode, n_devices=nd, warmup_steps=4, dtype="bf16")
    x0, _ = r.sample(x_T, plan, abar)     # capture
    x0, _ = r.sample(x_T, plan, abar)     # graph replay
    out[mode] = (x0, r.last_device_ms())
ref = out["reference"][0]
peak = float(ref.max() - ref.min())
rows = []
for mode, (x0, ms) in out.items():
    rel = float(np.linalg.norm((x0 - ref).ravel()) / np.linalg.norm(ref.ravel()))
    ps = A.psnr(x0, ref, peak)
    rows.append({"mode": mode, "bands": 1 if mode == "reference" else n, "rel_l2_vs_reference": rel,
                 "psnr_db": None if math.isinf(ps) else ps, "device_ms": ms})
    print(f"{mode:10s} bands={rows[-1]['bands']} rel-L2 {rel:.3e} PSNR {ps:6.2f} dB  {ms:8.2f} ms", flush=True)
json.dump(rows, open(os.environ.get("ABL_OUT", "gpurun_out/ablation.json"), "w"), indent=1)

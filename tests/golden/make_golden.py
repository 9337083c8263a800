"""Generate the committed golden fixtures from the reference's own CPU path.

Runs ONLY where /root/reference exists (it builds oracle/_ref from the unmodified
reference sources).  The fixtures pin the numpy oracle and the product's host logic on
machines without the reference (e.g. the GPU box).

  python tests/golden/make_golden.py        # writes tests/golden/reference_golden.npz
"""
from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import ref as R  # noqa: E402

TOY = (4, 16, 3, 4, 8, -1)         # ModelConfig defaults (model.hpp:30-36)
TINY = (2, 8, 2, 4, 8, -1)         # proj/tests/test_runtime.cpp:16-24
SDXL = (4, 320, 3, 32, 2048, -1)   # SURVEY.md §8 "SDXL-shape"


def main():
    out = {}
    # golden forward (proj/tests/test_model.cpp:234-246)
    m = R.Model(TOY, 42)
    y = m.forward_full(np.zeros((1, 4, 16, 16), np.float32), 10, np.zeros(8, np.float32))
    out["golden_forward"] = y
    # all layer outputs of a random forward (toy, 16x16, t=700)
    x = R.random_normal(1, 4, 16, 16, 79)
    cond = R.random_condition(8, 78)
    m77 = R.Model(TOY, 77)
    outs = m77.forward_collect(x, 700, cond)
    out["toy_collect_x"] = x
    out["toy_collect_cond"] = cond
    for i, o in enumerate(outs):
        out[f"toy_collect_{i:02d}"] = o
    # BASELINE config 1 (toy, 32x32, 4 steps, 2 patches) in every mode, with trajectories
    for mode, n, wu in [("reference", 1, 4), ("sync-pp", 2, 4), ("displaced", 2, 0),
                        ("displaced", 2, 1), ("naive", 2, 4), ("displaced", 4, 1)]:
        r = R.run_sampling(TOY, mode, n, 32, 32, 4, wu, trajectory=True)
        key = f"c1_{mode}_n{n}_w{wu}"
        out[key + "_x0"] = r["x0"]
        out[key + "_traj"] = r["trajectory"]
        out[key + "_macs"] = np.array([r["total_macs"]], dtype=np.uint64)
        out[key + "_vol"] = np.array(r["volumes"], dtype=np.uint64)
    # SDXL-shape: one reference forward on a 16x16 latent (weights from seed 42)
    ms = R.Model(SDXL, 42)
    xs = R.random_normal(1, 4, 16, 16, 1234)
    cs = R.random_condition(2048, 7)
    out["sdxl16_x"] = xs
    out["sdxl16_eps"] = ms.forward_full(xs, 980, cs)
    out["sdxl_weight_sha256"] = np.array(hashlib.sha256(
        np.concatenate([w.reshape(-1) for w in ms.weights()]).tobytes()).hexdigest())
    # patch specs (integer logic) for the BASELINE geometries
    specs = []
    for cfg, h, w, n in [(SDXL, 128, 128, 8), (SDXL, 160, 240, 8), (SDXL, 256, 256, 8),
                         (SDXL, 480, 480, 8), (TOY, 48, 48, 4), (TINY, 16, 16, 8)]:
        mm = R.Model(cfg, 1)
        for reg in R.partition_rows(h, n, w):
            lin, lout = mm.patch_spec(reg)
            specs.append(np.concatenate([np.array(list(cfg) + [h, w, n] + list(reg)), lin.reshape(-1),
                                         lout.reshape(-1)]))
    out["patch_specs"] = np.array(specs, dtype=object)
    # schedule / plan / DDIM (sampler.cpp)
    out["abar"] = R.make_schedule()
    out["plan50"] = np.array(R.make_plan(1000, 50))
    out["plan4"] = np.array(R.make_plan(1000, 4))
    np.savez_compressed(os.path.join(HERE, "reference_golden.npz"), **out)
    print("wrote", os.path.join(HERE, "reference_golden.npz"), len(out), "arrays")


if __name__ == "__main__":
    main()

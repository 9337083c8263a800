"""Bisect deeper-graph options: one reference-mode step per variant, finite check + oracle rel-L2."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import dataclasses  # noqa: E402

import numpy as np  # noqa: E402

from oracle import patchsim_np as O  # noqa: E402
from paper_2402_19481_b200 import patchsim as P  # noqa: E402

VARIANTS = [dict(res_blocks=2), dict(attn_depth=2), dict(attn_levels=0b110), dict(attn_levels=0b010),
            dict(attn_levels=0b110, attn_up=1), dict(attn_levels=0b011),
            dict(res_blocks=2, attn_depth=2), dict(res_blocks=2, attn_levels=0b110),
            dict(attn_depth=2, attn_levels=0b110), dict(res_blocks=2, attn_levels=0b110, attn_depth=2, attn_up=1)]
for kw in VARIANTS[int(sys.argv[1]) if len(sys.argv) > 1 else 0:]:
    cfg = dataclasses.replace(P.ModelConfig(), **kw)
    ocfg = O.ModelConfig(*[getattr(cfg, f) for f in ("in_channels", "base_channels", "levels", "groups",
                                                      "cond_dim", "attn_at_level", "res_blocks",
                                                      "attn_levels", "attn_depth", "attn_up")])
    m = P.build_model(cfg, 42)
    cond = O.random_condition(cfg.cond_dim, 7)
    x = O.random_normal(1, 4, 32, 32, 1234)
    for dt in ("fp32", "bf16"):
        r = P.PatchRunner(m, cond, 32, 32, mode="reference", dtype=dt)
        try:
            e = r.run_step(x, 700, 0)
            om = O.build_model(ocfg, 42)
            ref = O.forward_full(om, x, 700, cond)
            print(kw, dt, "finite", bool(np.isfinite(e).all()), "rel", O.rel_l2(e, ref), flush=True)
            r2 = P.PatchRunner(m, cond, 32, 32, mode="reference", dtype=dt)
            x0, _ = r2.sample(x, O.make_plan(1000, 3), O.make_schedule())
            print("   sample finite", bool(np.isfinite(x0).all()), flush=True)
        except Exception as ex:  # noqa: BLE001
            print(kw, dt, "ERR", str(ex)[:120], flush=True)

"""Fused conv + GroupNorm apply vs conv (+stats) + separate GN pass, per shape."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from gemm_micro import run, GN  # noqa: E402
from paper_2402_19481_b200 import _native as N  # noqa: E402

FUSED = 1 << 30
for name, kind, m, w, k, n, pix in [("L01", 1, 128, 128, 320, 320, 16384), ("L11", 1, 64, 64, 640, 640, 4096),
                                    ("L21", 1, 32, 32, 1280, 1280, 1024)]:
    plain = run(kind, m, w, k, n, reps=20)
    g = run(kind, m, w, k, n, reps=20 | GN)
    f = run(kind, m, w, k, n, reps=20 | FUSED)
    out = np.zeros(2)
    N.check(N.lib().pp_dev_gn_bench(0, pix, n, 32, 3, 50, out.ctypes.data_as(C.c_void_p)))
    extra = ""
    for tag, dbg in (("nowait", 32), ("nocoef", 64), ("nopass2", 128), ("none", 224)):
        x = run(kind, m, w, k, n, reps=20 | FUSED | (dbg << 22))
        extra += f" | {tag} {x[0]*1e3:6.1f}"
    print(extra)
    print(f"{name}: conv {plain[0]*1e3:6.1f} | conv+stats {g[0]*1e3:6.1f} (bn={int(g[1])} grid={int(g[4])}) + gn_apply "
          f"{out[0]:5.1f} = {g[0]*1e3 + out[0]:6.1f} | fused {f[0]*1e3:6.1f} (bn={int(f[1])} sp={int(f[2])} grid={int(f[4])})",
          flush=True)

"""Micro-benchmark of the GroupNorm apply / stats kernels on the SDXL-shape band sizes."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2402_19481_b200 import _native as N  # noqa: E402

for name, pix, c, flags in [("128^2 x 320 silu+temb", 16384, 320, 3), ("128^2 x 320 silu+temb+skip", 16384, 320, 7),
                            ("64^2 x 640 silu+temb", 4096, 640, 3), ("32^2 x 1280 silu+temb", 1024, 1280, 3),
                            ("128^2 x 320 silu (head)", 16384, 320, 1),
                            ("128^2 x 320 silu+temb+skip +stats", 16384, 320, 15)]:
    out = np.zeros(2)
    N.check(N.lib().pp_dev_gn_bench(0, pix, c, 32, flags, 50, out.ctypes.data_as(C.c_void_p)))
    mb = pix * c * 2 * (3 if flags & 4 else 2) / 1e6
    print(f"{name:30s} apply {out[0]:6.2f} us ({mb / out[0]:5.2f} TB/s)  stats {out[1]:6.2f} us", flush=True)

"""MMA issue-loop cost: mmaOnly vs mmaOnly without full-barrier waits (bit 16), per bn."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2402_19481_b200 import _native as N  # noqa: E402

M, K = 2 * 148 * 128, 2880
for bn in (64, 160, 256):
    for cta in (32, 16):
        line = f"{'pair' if cta == 16 else 'single':6s} bn={bn:3d}"
        for mode, bits in (("mmaOnly", 6), ("mmaOnly+nowait", 6 | 16), ("noMMA,noEpi", 5),
                           ("nothing", 7), ("nothing+nowait", 7 | 16)):
            out = np.zeros(5)
            N.check(N.lib().pp_dev_gemm_bench(0, 0, M, 1, K, bn, 1 | cta, bn, 20 | (bits << 22),
                                              out.ctypes.data_as(C.c_void_p)))
            line += f" | {mode} {out[0] * 1e6 / 90:6.1f} ns/kb"
        print(line, flush=True)

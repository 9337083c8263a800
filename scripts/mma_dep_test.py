"""MMA issue-path cost per 128-byte K block (exact waves): MMA-only vs full kernel."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2402_19481_b200 import _native as N  # noqa: E402

M, K = 2 * 148 * 128, 2880
for bn in (64, 128, 160, 256):
    for name, bits in (("mmaOnly", 6), ("noEpi", 4), ("full", 0)):
        out = np.zeros(5)
        N.check(N.lib().pp_dev_gemm_bench(0, 0, M, 1, K, bn, 1, bn, 20 | (bits << 22),
                                          out.ctypes.data_as(C.c_void_p)))
        tf = 2.0 * M * bn * K / (out[0] * 1e-3) / 1e12
        print(f"bn={bn:3d} {name:8s} {out[0] * 1e6 / (2 * K // 64):7.1f} ns/kblock {tf:7.1f} TF/s",
              flush=True)

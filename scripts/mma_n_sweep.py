"""MMA-only cost per 128-byte K block vs MMA N (no TMA, no epilogue), exact waves.

M = 2 * 148 * 128 rows -> every CTA runs exactly 2 tiles of 45 K blocks (per n-tile).
"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2402_19481_b200 import _native as N  # noqa: E402

M, K = 2 * 148 * 128, 2880
for bn in (64, 96, 128, 160, 192, 224, 256):
  for cta in (32, 16):
    for mode, bits in (("mmaOnly", 6), ("full", 0), ("noEpi", 4)):
        out = np.zeros(5)
        N.check(N.lib().pp_dev_gemm_bench(0, 0, M, 1, K, bn, 1 | cta, bn, 20 | (bits << 22),
                                          out.ctypes.data_as(C.c_void_p)))
        us = out[0] * 1e3
        kb = 2 * (K // 64)
        tf = 2.0 * M * bn * K / (out[0] * 1e-3) / 1e12
        print(f"{'pair' if cta == 16 else 'single':6s} bn={bn:3d} {mode:8s} {us:8.2f} us  "
              f"{us * 1e3 / kb:7.1f} ns/kblock  {tf:7.1f} TF/s", flush=True)

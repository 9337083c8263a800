"""Fixed cost of the tcgen05 GEMM kernel: mean us per launch (back to back, CUDA events) of
small shapes whose work is negligible, with and without PDL (PP_PDL env, read at load), and
-- in a -DPP_GEMM_DEBUG build -- with the kernel's debug flags (1 no MMA, 2 no TMA, 4 no
epilogue) to split the skeleton cost from the data path.

usage: [PP_PDL=0] [PP_B200_LIB=ab/lib_debug.so] python scripts/latency_micro.py [DEBUG_FLAGS...]
"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2402_19481_b200 import _native as N  # noqa: E402

GN = 1 << 20
SHAPES = [  # name, kind, M_or_rows, W, K, N, flags
    ("1 tile GEMM 128x64x16", 0, 128, 1, 64, 16, 0),
    ("148 tiles GEMM 18944x64x16", 0, 18944, 1, 64, 16, 0),
    ("stem GEMM 16384x64x320", 0, 16384, 1, 64, 320, 0),
    ("stem GEMM 16384x64x320 +gn", 0, 16384, 1, 64, 320, GN),
    ("head conv 320->4 @128^2", 1, 128, 128, 320, 4, 0),
    ("linear 1024x1280x1280", 0, 1024, 1, 1280, 1280, 0),
    ("L01 conv 320->320 @128^2", 1, 128, 128, 320, 320, 0),
    ("L01 conv 320->320 @128^2 +gn", 1, 128, 128, 320, 320, GN),
]
dbgs = [int(x) for x in sys.argv[1:]] or [0]
print(f"PDL={os.environ.get('PP_PDL', '1')} lib={os.path.basename(N.LIB_PATH)}")
for name, kind, m, w, k, n, fl in SHAPES:
    line = f"{name:32s}"
    for d in dbgs:
        out = np.zeros(5)
        N.check(N.lib().pp_dev_gemm_bench(0, kind, m, w, k, n, 0, 0, 50 | fl | (d << 22),
                                          out.ctypes.data_as(C.c_void_p)))
        line += f"  dbg{d}: {out[0] * 1e3:7.2f} us"
    print(line + f"  (bn={int(out[1])} grid={int(out[4])} stages={int(out[3])})")

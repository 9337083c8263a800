"""Cost of the parts of the fused GroupNorm-statistics conv epilogue (a -DPP_GEMM_DEBUG build
with skip flags: 8 column sums, 16 per-tile section, 32 fold, 64 relaxed ticket; 4 no epilogue).
usage: PP_B200_LIB=ab/lib_debug.so python scripts/gn_epilogue_parts.py"""
import ctypes as C, os, sys
import numpy as np
sys.path.insert(0, os.getcwd())
from paper_2402_19481_b200 import _native as N
GN = 1 << 20
for name, kind, m, w, k, n in [("L01 conv 320 @128^2", 1, 128, 128, 320, 320), ("L11 conv 640 @64^2", 1, 64, 64, 640, 640),
                               ("L21 conv 1280 @32^2", 1, 32, 32, 1280, 1280), ("stem GEMM", 0, 16384, 1, 64, 320)]:
    line = f"{name:24s}"
    for lab, fl, d in [("nogn", 0, 0), ("gn", GN, 0), ("gn-nochunk", GN, 8), ("gn-nosect", GN, 16), ("gn-nofold", GN, 32), ("gn-none", GN, 24), ("gn-relaxed", GN, 64), ("noepi", GN, 4)]:
        out = np.zeros(5)
        N.check(N.lib().pp_dev_gemm_bench(0, kind, m, w, k, n, 0, 0, 50 | fl | (d << 22), out.ctypes.data_as(C.c_void_p)))
        line += f" {lab}:{out[0]*1e3:6.2f}"
    print(line, flush=True)

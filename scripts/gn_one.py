"""One GroupNorm-pass configuration (for ncu): python scripts/gn_one.py PIX C FLAGS"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2402_19481_b200 import _native as N  # noqa: E402

pix, c, flags = (int(v) for v in sys.argv[1:4])
out = np.zeros(2)
N.check(N.lib().pp_dev_gn_bench(0, pix, c, 32, flags, 3, out.ctypes.data_as(C.c_void_p)))
print(out)

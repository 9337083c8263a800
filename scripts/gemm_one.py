"""Run one GEMM/conv configuration of the tcgen05 kernel (for ncu captures).

usage: python scripts/gemm_one.py KIND M_OR_ROWS W K N FORCE BN [REPS]
  KIND 0 = GEMM, 1/2 = conv stride 1/2; FORCE = force_splits bits (16 pair, 32 single)
Prints mean us per launch (meaningless under ncu)."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2402_19481_b200 import _native as N  # noqa: E402

kind, m, w, k, n, force, bn = (int(x) for x in sys.argv[1:8])
reps = int(sys.argv[8]) if len(sys.argv) > 8 else 2
out = np.zeros(5)
N.check(N.lib().pp_dev_gemm_bench(0, kind, m, w, k, n, force, bn, reps, out.ctypes.data_as(C.c_void_p)))
print(f"{out[0] * 1e3:.1f} us bn={int(out[1])} splits={int(out[2])} stages={int(out[3])} grid={int(out[4])}")

"""Where the time of the small head/stem convs goes (L00 4->320, L62 320->4 at 128^2)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from gemm_micro import run  # noqa: E402

VAR = [("full", 0), ("noMMA", 1), ("noTMA", 2), ("noEpi", 4), ("mmaOnly", 6), ("tmaOnly", 5)]
for name, kind, m, w, k, n in [("L00 4(64)->320", 1, 128, 128, 64, 320), ("L62 320->4", 1, 128, 128, 320, 4)]:
    line = name
    for vn, dbg in VAR:
        o = run(kind, m, w, k, n, reps=20 | (dbg << 22))
        line += f" | {vn} {o[0] * 1e3:6.1f}"
    line += f" (bn={int(o[1])} sp={int(o[2])} st={int(o[3])} grid={int(o[4])})"
    print(line, flush=True)

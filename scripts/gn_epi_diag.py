"""Cost of the fused GroupNorm-statistics epilogue parts (debug bits 32/64/128)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from gemm_micro import run, GN  # noqa: E402

for name, kind, m, w, k, n in [("L01", 1, 128, 128, 320, 320), ("L11", 1, 64, 64, 640, 640),
                               ("L37", 1, 64, 64, 1280, 640), ("L21", 1, 32, 32, 1280, 1280)]:
    line = f"{name}"
    for vn, flags in [("nogn", 0), ("gn", GN), ("gn-butterfly", GN | (32 << 22)),
                      ("gn-tilefold", GN | (64 << 22)), ("gn-final", GN | (128 << 22)),
                      ("gn-all3", GN | (224 << 22))]:
        o = run(kind, m, w, k, n, reps=20 | flags)
        line += f" | {vn} {o[0] * 1e3:6.1f}"
    print(line, flush=True)

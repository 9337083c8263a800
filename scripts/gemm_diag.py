"""Diagnose the tcgen05 conv kernel: {single, pair} x {full, noMMA, noTMA, noEpi, mmaOnly, tmaOnly}."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from gemm_micro import run, flops, PAIR, SINGLE  # noqa: E402

SH = [("L01 128^2 320->320", 1, 128, 128, 320, 320, 160, 1),
      ("L11 64^2 640->640", 1, 64, 64, 640, 640, 160, 1),
      ("L37 64^2 1280->640", 1, 64, 64, 1280, 640, 160, 1),
      ("L21 32^2 1280->1280", 1, 32, 32, 1280, 1280, 160, 2)]
VAR = [("full", 0), ("noMMA", 1), ("noTMA", 2), ("noEpi", 4), ("mmaOnly", 6), ("tmaOnly", 5)]
for name, kind, m, w, k, n, bn, sp in SH:
    for cta, cn in ((SINGLE, "single"), (PAIR, "pair")):
        line = f"{name:22s} {cn:6s} bn={bn} sp={sp}"
        for vn, dbg in VAR:
            o = run(kind, m, w, k, n, sp | cta, bn, reps=20 | (dbg << 22))
            line += f" | {vn} {o[0] * 1e3:6.1f}"
        o = run(kind, m, w, k, n, sp | cta, bn)
        line += f" | {flops(kind, m, w, k, n) / (o[0] * 1e-3) / 1e12:6.0f} TF/s st={int(o[3])} grid={int(o[4])}"
        print(line, flush=True)

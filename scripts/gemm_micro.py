"""Micro-benchmark of the tcgen05 GEMM / implicit-conv kernel on the SDXL-shape layer shapes.

usage (GPU box): python scripts/gemm_micro.py [--sweep] [--variants]
Prints TFLOP/s per shape (mean of launches, CUDA events).  --variants adds the fused
GroupNorm-statistics epilogue and a cold L2 (256 MiB flush before each launch).
"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2402_19481_b200 import _native as N  # noqa: E402

# (name, kind, M_or_rows, W, K(=C_in), N) -- 1024^2 SDXL-shape conv layers at N=1 (Appendix A)
SHAPES = [
    ("L01 conv 320->320 @128^2", 1, 128, 128, 320, 320),
    ("L49 conv 640->320 @128^2", 1, 128, 128, 640, 320),
    ("L10 down 320->640 @128^2", 2, 128, 128, 320, 640),
    ("L11 conv 640->640 @64^2", 1, 64, 64, 640, 640),
    ("L37 conv 1280->640 @64^2", 1, 64, 64, 1280, 640),
    ("L21 conv 1280->1280 @32^2", 1, 32, 32, 1280, 1280),
    ("L01/8 band 320->320 16x128", 1, 16, 128, 320, 320),
    ("L11/8 band 640->640 8x64", 1, 8, 64, 640, 640),
    ("L21/8 band 1280 4x32", 1, 4, 32, 1280, 1280),
    ("GEMM 16384x320x2880", 0, 16384, 1, 2880, 320),
    ("GEMM 8192x8192x8192", 0, 8192, 1, 8192, 8192),
]
GN, FLUSH, NOCLUSTER = 1 << 20, 1 << 21, 1 << 30
PAIR, SINGLE = 16, 32   # force_splits flag bits: CTA-pair / single-CTA kernel


def flops(kind, m, w, k, n):
    if kind == 0:
        return 2.0 * m * n * k
    pix = (m * w) if kind == 1 else (m // 2) * (w // 2)
    return 2.0 * pix * n * 9 * k


def run(kind, m, w, k, n, splits=0, bn=0, reps=20):
    out = np.zeros(5)
    N.check(N.lib().pp_dev_gemm_bench(0, kind, m, w, k, n, splits, bn, reps,
                                      out.ctypes.data_as(C.c_void_p)))
    return out


def main():
    sweep = "--sweep" in sys.argv
    variants = "--variants" in sys.argv
    for name, kind, m, w, k, n in SHAPES:
        o = run(kind, m, w, k, n)
        tf = flops(kind, m, w, k, n) / (o[0] * 1e-3) / 1e12
        line = (f"{name:30s} {o[0] * 1e3:8.1f} us {tf:7.1f} TF/s  bn={int(o[1])} "
                f"splits={int(o[2])} stages={int(o[3])} grid={int(o[4])}")
        if kind != 0:
            g = run(kind, m, w, k, n, reps=20 | GN)
            line += f" | +gn {g[0] * 1e3:7.1f} us"
        if "--cluster" in sys.argv:
            g = run(kind, m, w, k, n, reps=20 | GN) if kind else o
            c1 = run(kind, m, w, k, n, reps=20 | NOCLUSTER)
            g1 = run(kind, m, w, k, n, reps=20 | GN | NOCLUSTER) if kind else c1
            line += (f" | +gn {g[0] * 1e3:7.1f} us | cluster1 {c1[0] * 1e3:7.1f} us "
                     f"(grid {int(c1[4])}) +gn {g1[0] * 1e3:7.1f} us")
        if variants and kind != 0:
            g = run(kind, m, w, k, n, reps=20 | GN)
            c = run(kind, m, w, k, n, reps=10 | GN | FLUSH)
            nm = run(kind, m, w, k, n, reps=20 | (1 << 22))
            nt = run(kind, m, w, k, n, reps=20 | (2 << 22))
            ne = run(kind, m, w, k, n, reps=20 | (4 << 22))
            nb = run(kind, m, w, k, n, reps=20 | (6 << 22))
            bo = run(kind, m, w, k, n, reps=20 | ((4 | 64) << 22))
            ao = run(kind, m, w, k, n, reps=20 | ((4 | 128) << 22))
            line += (f" | +gn {g[0] * 1e3:7.1f} us | +gn+coldL2 {c[0] * 1e3:7.1f} us"
                     f" | noMMA {nm[0] * 1e3:7.1f} us | noTMA {nt[0] * 1e3:7.1f} us"
                     f" | noEpi {ne[0] * 1e3:7.1f} us | mmaOnly {nb[0] * 1e3:7.1f} us"
                     f" | noEpi+Bonly {bo[0] * 1e3:7.1f} us | noEpi+Aonly {ao[0] * 1e3:7.1f} us")
        print(line, flush=True)
        if "--cta" in sys.argv:
            for cta, nm in ((SINGLE, "single"), (PAIR, "pair")):
                for bn in (128, 160, 256):
                    if n % bn:
                        continue
                    for sp in (1, 2):
                        try:
                            o = run(kind, m, w, k, n, sp | cta, bn)
                        except Exception as e:  # noqa: BLE001
                            print("   ", nm, bn, sp, "ERR", e)
                            continue
                        tf = flops(kind, m, w, k, n) / (o[0] * 1e-3) / 1e12
                        print(f"    {nm:6s} bn={bn:3d} splits={sp}  {o[0] * 1e3:8.1f} us "
                              f"{tf:7.1f} TF/s stages={int(o[3])} grid={int(o[4])}", flush=True)
        if sweep and kind != 0:
            for bn in (64, 128, 160, 256):
                if n % bn:
                    continue
                for sp in (1, 2):
                    try:
                        o = run(kind, m, w, k, n, sp, bn)
                    except Exception as e:  # noqa: BLE001
                        print("   ", bn, sp, "ERR", e)
                        continue
                    tf = flops(kind, m, w, k, n) / (o[0] * 1e-3) / 1e12
                    print(f"    bn={bn:3d} splits={sp}  {o[0] * 1e3:8.1f} us {tf:7.1f} TF/s "
                          f"stages={int(o[3])}", flush=True)


if __name__ == "__main__":
    main()

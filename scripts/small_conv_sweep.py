"""Tiling sweep of the small head/stem convs (L00 4->320, L62 320->4 at 128^2): the planner's
choice against forced splits / CTA pairs / block_n (force bits: 1-2 splits, 16 pair, 32 single)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from gemm_micro import run  # noqa: E402

for name, kind, m, w, k, n, bns in [("L62 320->4", 1, 128, 128, 320, 4, [0]),
                                     ("L00 4(64)->320", 1, 128, 128, 64, 320, [0, 32, 64, 80, 160, 320])]:
    for force in (0, 2, 16, 18, 32, 34):
        for bn in bns:
            try:
                o = run(kind, m, w, k, n, splits=force, bn=bn, reps=50)
            except Exception as e:  # noqa: BLE001
                print(f"{name} force={force} bn={bn}: {e}")
                continue
            print(f"{name:16s} force={force:2d} bn={bn:3d} -> {o[0] * 1e3:6.1f} us (bn={int(o[1])} "
                  f"sp={int(o[2])} st={int(o[3])} grid={int(o[4])})", flush=True)

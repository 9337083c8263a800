"""Wide tile (block_n = 320, two N-half MMAs) vs block_n = 160 on the N = 320 / 640 conv shapes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from gemm_micro import run, GN, SINGLE, PAIR  # noqa: E402

for name, kind, m, w, k, n in [("L01 128^2 320", 1, 128, 128, 320, 320), ("L49 128^2 640->320", 1, 128, 128, 640, 320),
                               ("L11 64^2 640", 1, 64, 64, 640, 640), ("L37 64^2 1280->640", 1, 64, 64, 1280, 640)]:
    line = name
    for tag, force, bn in (("auto", 0, 0), ("s160", SINGLE | 1, 160), ("p160", PAIR | 1, 160), ("s320", SINGLE | 1, 320), ("p320", PAIR | 1, 320)):
        try:
            o = run(kind, m, w, k, n, force, bn)
            g = run(kind, m, w, k, n, force, bn, reps=20 | GN)
            line += f" | {tag} {o[0] * 1e3:6.1f} gn {g[0] * 1e3:6.1f} (bn={int(o[1])} st={int(o[3])} grid={int(o[4])})"
        except Exception as e:  # noqa: BLE001
            line += f" | {tag} ERR {e}"
    print(line, flush=True)

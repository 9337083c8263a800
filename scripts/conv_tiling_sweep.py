"""Tiling sweep of the parallelism-starved SDXL-shape convs at 1024^2 (32^2 layers, the
DownConvs): the planner's choice against forced splits / pair / block_n.
FORCES / BNS env: comma lists (force bits: 1-2 splits, 16 pair, 32 single)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from gemm_micro import run  # noqa: E402

SHAPES = [("L21 32^2 1280->1280", 1, 32, 32, 1280, 1280), ("L20 down 640->1280", 2, 64, 64, 640, 1280),
          ("L10 down 320->640", 2, 128, 128, 320, 640), ("L37 64^2 1280->640", 1, 64, 64, 1280, 640)]
forces = [int(x) for x in os.environ.get("FORCES", "0,1,2,17,18,33,34").split(",")]
bns = [int(x) for x in os.environ.get("BNS", "0,64,80,128,160,256").split(",")]
for name, kind, m, w, k, n in SHAPES:
    for force in forces:
        for bn in bns:
            try:
                o = run(kind, m, w, k, n, splits=force, bn=bn, reps=30)
            except Exception as e:  # noqa: BLE001
                print(f"{name} force={force} bn={bn}: {str(e)[:60]}")
                continue
            print(f"{name:20s} force={force:2d} bn={bn:3d} -> {o[0] * 1e3:6.1f} us (bn={int(o[1])} "
                  f"sp={int(o[2])} st={int(o[3])} grid={int(o[4])})", flush=True)

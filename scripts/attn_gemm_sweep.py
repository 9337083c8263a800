"""Tiling sweep of the attention GEMMs at 1024^2 (S = Q K^T: M=1024 N=1024 K=1280; O = P V:
M=1024 N=1280 K=1024): the planner's choice against forced splits / pair / block_n."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from gemm_micro import run  # noqa: E402

for name, m, k, n in [("S=QK^T", 1024, 1280, 1024), ("O=PV", 1024, 1024, 1280),
                      ("L34 linear", 1024, 1280, 1280)]:
    forces = [int(x) for x in os.environ.get("FORCES", "0,2,16,18,32,34").split(",")]
    bns = [int(x) for x in os.environ.get("BNS", "0,64,128,256").split(",")]
    for force in forces:
        for bn in bns:
            try:
                o = run(0, m, 0, k, n, splits=force, bn=bn, reps=50)
            except Exception as e:  # noqa: BLE001
                print(f"{name} force={force} bn={bn}: {str(e)[:60]}")
                continue
            print(f"{name:10s} force={force:2d} bn={bn:3d} -> {o[0] * 1e3:6.1f} us (bn={int(o[1])} "
                  f"sp={int(o[2])} st={int(o[3])} grid={int(o[4])})", flush=True)

"""A/B the conv kernel of two builds (PP_B200_LIB) on the SDXL conv shapes: warm / +gn / +gn cold-L2."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from gemm_micro import SHAPES, run, GN, FLUSH  # noqa: E402

tag = os.environ.get("TAG", "new")
for name, kind, m, w, k, n in SHAPES[:6]:
    o = run(kind, m, w, k, n)
    g = run(kind, m, w, k, n, reps=20 | GN)
    c = run(kind, m, w, k, n, reps=10 | GN | FLUSH)
    print(f"{tag:4s} {name:28s} warm {o[0] * 1e3:6.1f} | +gn {g[0] * 1e3:6.1f} | +gn cold {c[0] * 1e3:6.1f} us",
          flush=True)

"""Per-tap check of the slab-mode conv: weights non-zero at one tap only."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2402_19481_b200 import _native as N  # noqa: E402


def _p(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


rows, W, Cc, co = 4, 128, 64, 128
g = torch.Generator(device="cuda").manual_seed(1)
inp = torch.randn(rows + 2, W, Cc, device="cuda", generator=g).bfloat16()
for tap in range(9):
    ky, kx = tap // 3, tap % 3
    w = torch.zeros(co, 3, 3, Cc, device="cuda")
    w[:, ky, kx, :] = torch.randn(co, Cc, device="cuda", generator=g) / 8
    w = w.bfloat16()
    bias = torch.zeros(co, device="cuda")
    out = torch.zeros(rows, W, co, device="cuda", dtype=torch.float32)
    N.check(N.lib().pp_dev_conv(0, _p(inp), rows, W, Cc, 1, _p(w), co, co, _p(bias), _p(out), co, 1,
                                None, 0, 32 | 1, 0, None))
    x = inp.double().permute(2, 0, 1).unsqueeze(0)
    ref = torch.nn.functional.conv2d(x, w.double().permute(0, 3, 1, 2), None, padding=(0, 1))[0].permute(1, 2, 0)
    err = ((out.double() - ref).norm() / ref.norm()).item()
    # where does the output match a shifted reference?
    best = None
    for dy in (-1, 0, 1):
        for dx in range(-8, 9):
            r2 = torch.roll(ref, shifts=(dy, dx), dims=(0, 1))
            e2 = ((out.double() - r2)[1:-1, 9:-9].norm() / r2[1:-1, 9:-9].norm()).item()
            if best is None or e2 < best[0]:
                best = (e2, dy, dx)
    print(f"tap {tap} (ky={ky},kx={kx}) off={ky * 130 + kx} err {err:.3e}  best shift {best}", flush=True)

"""GPU fp64 restatement of the reference path (torch), for parity at full benchmark sizes.

TEST INFRASTRUCTURE ONLY (like ``oracle/patchsim_np.py``): the product never imports it.

The numpy oracle (``oracle/patchsim_np.py``) is a line-by-line restatement of the
reference's CPU path, but at the benchmarked geometry (SDXL-shape, 128x128 latent and up)
one numpy step takes minutes.  This module re-executes that same source with the tensor
kernels replaced by torch float64 versions on a CUDA device, keeping everything else --
model builder, weight pool, patch specs, the PatchRunner's sync / displaced / naive step
logic, GroupNorm statistic combination, DDIM sampler -- literally the numpy oracle's code.
Arithmetic contract is the reference's (``proj/src/tensor.cpp``): fp32 storage, fp64
accumulation, one fp32 rounding per operator output; only the fp64 summation order differs,
so results agree with the numpy oracle to fp32 rounding (pinned in tests/test_oracle_torch.py
at small sizes and against the reference build, ``oracle/_ref``, at 128x128).

Usage:  T = load(device)  ->  module with the numpy oracle's API (T.run_sampling,
T.PatchRunner, T.forward_full, ...); step results come back as numpy float32.
"""
from __future__ import annotations

import importlib.util
import math
import sys

import numpy as np

from . import patchsim_np as _NP

_cache = {}


def load(device="cuda"):
    """A fresh instance of the numpy oracle module with torch fp64 kernels on `device`."""
    key = str(device)
    if key in _cache:
        return _cache[key]
    import torch
    import torch.nn.functional as F

    spec = importlib.util.spec_from_file_location("oracle._patchsim_torch_" + key.replace(":", "_"),
                                                  _NP.__file__)
    T = importlib.util.module_from_spec(spec)
    sys.modules[spec.name] = T
    spec.loader.exec_module(T)
    dev = torch.device(device)
    f32, f64 = torch.float32, torch.float64
    wcache = {}

    def t32(a):
        """host numpy / torch -> float32 tensor on the device."""
        if isinstance(a, torch.Tensor):
            return a.to(dev, f32)
        return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(dev)

    def w64(a):
        """weights (numpy arrays of the model pool, uploaded once) -> float64 tensor."""
        k = id(a)
        hit = wcache.get(k)
        if hit is not None and hit[0] is a:
            return hit[1]
        v = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(dev, f64)
        wcache[k] = (a, v)
        return v

    def conv2d_region(x, region, weight, bias, stride, pad):
        """tensor.cpp:79-130 (see patchsim_np.conv2d_region)."""
        x = t32(x)
        n, c, h, w = x.shape
        r0, r1 = region[0], region[1]
        if not (0 <= r0 < r1 <= h):
            raise T.InvalidArgument(f"conv2d_region: invalid region [{r0},{r1}) of {h}x{w}")
        co, ci, k, _ = weight.shape
        if ci != c:
            raise T.InvalidArgument(f"conv2d: weight expects c_in={ci}, input has c={c}")
        out_h = (h + 2 * pad - k) // stride + 1
        oy0 = min(-(-r0 // stride), out_h)
        oy1 = min(-(-r1 // stride), out_h)
        if oy0 >= oy1:
            raise T.InvalidArgument("conv2d_region: region maps to no output rows")
        iy_lo = oy0 * stride - pad
        iy_hi = (oy1 - 1) * stride - pad + k
        xp = torch.zeros((n, c, iy_hi - iy_lo, w), dtype=f64, device=dev)
        lo, hi = max(iy_lo, 0), min(iy_hi, h)
        xp[:, :, lo - iy_lo:hi - iy_lo, :] = x[:, :, lo:hi, :].to(f64)
        acc = F.conv2d(xp, w64(weight), None, stride=stride, padding=(0, pad))
        acc = acc + w64(bias).reshape(1, -1, 1, 1)
        return acc.to(f32)

    def linear(tokens, weight, bias):
        tokens = t32(tokens)
        n, _, t, i = tokens.shape
        o = weight.shape[0]
        acc = tokens.reshape(n * t, i).to(f64) @ w64(weight).reshape(o, i).T
        acc = acc + w64(bias).reshape(-1)
        return acc.to(f32).reshape(n, 1, t, o)

    def attention(q, k, v, scale):
        """tensor.cpp:163-199: softmax(q k^T scale) v in fp64 with the row max subtracted."""
        q, k, v = t32(q), t32(k), t32(v)
        out = torch.empty((q.shape[0], 1, q.shape[2], v.shape[3]), dtype=f32, device=dev)
        sc = float(np.float32(scale))
        for b in range(q.shape[0]):
            lg = (q[b, 0].to(f64) @ k[b, 0].to(f64).T) * sc
            lg = torch.exp(lg - lg.max(dim=1, keepdim=True).values)
            den = lg.sum(dim=1, keepdim=True)
            out[b, 0] = ((lg @ v[b, 0].to(f64)) / den).to(f32)
        return out

    def group_stats(x, groups, region=None):
        x = t32(x)
        n, c, h, w = x.shape
        if groups <= 0 or c % groups:
            raise T.InvalidArgument(f"group_stats: channels {c} not divisible by groups {groups}")
        y0, y1 = (0, h) if region is None else (region[0], region[1])
        v = x[:, :, y0:y1, :].to(f64).reshape(n, groups, -1)
        cnt = float(c // groups) * (y1 - y0) * w
        mu = (v.sum(dim=2) / cnt).reshape(-1).cpu().numpy()
        msq = ((v * v).sum(dim=2) / cnt).reshape(-1).cpu().numpy()
        return mu, msq

    def group_norm_apply(x, region, mean, mean_sq, gamma, beta, eps):
        x = t32(x)
        n, c, h, w = x.shape
        groups = len(mean) // n
        var = np.asarray(mean_sq) - np.asarray(mean) * np.asarray(mean)
        if np.any(var < 0.0):
            raise T.RuntimeFailure(
                "group_norm_apply: negative variance (caller must substitute fallback stats)")
        inv_std = 1.0 / np.sqrt(var + float(np.float32(eps)))
        y0, y1 = (0, h) if region is None else (region[0], region[1])
        cpg = c // groups
        mu = torch.from_numpy(np.repeat(np.asarray(mean).reshape(n, groups), cpg, axis=1)).to(dev)
        isd = torch.from_numpy(np.repeat(inv_std.reshape(n, groups), cpg, axis=1)).to(dev)
        g = w64(gamma).reshape(1, c, 1, 1)
        b = w64(beta).reshape(1, c, 1, 1)
        out = x.clone()
        seg = x[:, :, y0:y1, :].to(f64)
        out[:, :, y0:y1, :] = ((seg - mu[:, :, None, None]) * isd[:, :, None, None] * g + b).to(f32)
        return out

    def scatter_region(stale_full, fresh, region):
        out = t32(stale_full).clone()
        fresh = t32(fresh)
        out[:, :, region[0]:region[0] + fresh.shape[2], :] = fresh
        return out

    def silu(x):
        v = t32(x).to(f64)
        return (v / (1.0 + torch.exp(-v))).to(f32)

    def add(x, y):
        x, y = t32(x), t32(y)
        if x.shape != y.shape:
            raise T.InvalidArgument(f"add: shape mismatch {tuple(x.shape)} vs {tuple(y.shape)}")
        return x + y

    def upsample_nearest2x(x):
        x = t32(x)
        return x.repeat_interleave(2, dim=2).repeat_interleave(2, dim=3)

    def to_tokens(x):
        x = t32(x)
        n, c, h, w = x.shape
        return x.reshape(n, c, h * w).transpose(1, 2).reshape(n, 1, h * w, c)

    def from_tokens(t, c, h, w):
        return t.reshape(t.shape[0], h * w, c).transpose(1, 2).reshape(t.shape[0], c, h, w).contiguous()

    def layer_time_emb(m, d, x, emb):
        p = T.time_projection(m, d, emb)
        return t32(x) + t32(p).reshape(1, -1, 1, 1)

    def all_finite(x):
        if isinstance(x, torch.Tensor):
            return bool(torch.isfinite(x).all())
        return bool(np.all(np.isfinite(x)))

    def cat_rows(parts):
        return torch.cat([t32(p) for p in parts], dim=2)

    def rows(x, a, b):
        return t32(x)[:, :, a:b, :].clone()

    def host(x):
        if isinstance(x, torch.Tensor):
            return x.detach().to("cpu", f32).numpy()
        return x

    for name, fn in dict(conv2d_region=conv2d_region, linear=linear, attention=attention,
                         group_stats=group_stats, group_norm_apply=group_norm_apply,
                         scatter_region=scatter_region, silu=silu, add=add,
                         upsample_nearest2x=upsample_nearest2x, to_tokens=to_tokens,
                         from_tokens=from_tokens, layer_time_emb=layer_time_emb,
                         _all_finite=all_finite, _cat_rows=cat_rows, _rows=rows,
                         _host=host).items():
        setattr(T, name, fn)
    T.DEVICE = dev
    T.to_host = host
    _cache[key] = T
    return T


def rel_l2(a, b):
    return _NP.rel_l2(a, b)


__all__ = ["load", "rel_l2", "math"]

"""Kernel-level operators on the B200 vs the CPU oracle (restating proj/tests/test_tensor.cpp).

Each operator goes through the C ABI (pp_conv2d_region, pp_linear, pp_attention,
pp_group_stats, pp_group_norm_apply, pp_silu, pp_upsample_nearest2x, pp_ddim_update),
i.e. through the same sm_100a kernels as the runner.  Tolerances: fp32 mode = TF32 tensor
cores (inputs rounded to a 10-bit mantissa) -> rel-L2 <= 1e-3; bf16 mode -> <= 1e-2.
"""
import ctypes as C

import numpy as np
import pytest

from oracle import patchsim_np as O
from paper_2402_19481_b200 import _native as N

pytestmark = pytest.mark.gpu
TOL = {"fp32": 1e-3, "bf16": 1e-2}


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def conv(dtype, x, region, w, b, stride):
    x, w, b = f32(x), f32(w), f32(b)
    n, c, h, wd = x.shape
    co = w.shape[0]
    out_h = (h + 2 - 3) // stride + 1
    out_w = (wd + 2 - 3) // stride + 1
    oy0 = min(-(-region[0] // stride), out_h)
    oy1 = min(-(-region[1] // stride), out_h)
    out = np.zeros((n, co, oy1 - oy0, out_w), np.float32)
    N.check(N.lib().pp_conv2d_region(N.DTYPES[dtype], _p(x), n, c, h, wd, region[0], region[1],
                                     _p(w), co, 3, _p(b), stride, 1, _p(out)))
    return out


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
def test_conv_identity_zero_and_ramp(dtype):
    # test_tensor.cpp:43-71: identity-center kernel, zero weights -> bias, 45-sum ramp
    x = np.ones((1, 1, 3, 3), np.float32)
    w = np.zeros((1, 1, 3, 3), np.float32)
    w[0, 0, 1, 1] = 1
    assert np.array_equal(conv(dtype, x, (0, 3), w, np.zeros(1), 1), x)
    xr = O.random_normal(1, 3, 5, 5, 7)
    y = conv(dtype, xr, (0, 5), np.zeros((2, 3, 3, 3)), np.array([0.25, -1.5]), 1)
    assert np.all(y[0, 0] == 0.25) and np.all(y[0, 1] == -1.5)
    ramp = np.arange(9, dtype=np.float32).reshape(1, 1, 3, 3)
    y = conv(dtype, ramp, (0, 3), np.ones((1, 1, 3, 3)), np.zeros(1), 1)
    assert y[0, 0, 1, 1] == 36 and y[0, 0, 0, 0] == 8   # sums of the padded 3x3 windows


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
@pytest.mark.parametrize("stride,shape,region", [
    (1, (1, 5, 9, 7), (0, 9)), (1, (2, 16, 12, 10), (3, 7)), (2, (1, 8, 12, 12), (4, 8)),
    (2, (1, 6, 9, 7), (2, 9)), (1, (1, 64, 32, 32), (8, 16)), (2, (1, 64, 32, 32), (0, 32))])
def test_conv_region_vs_oracle(dtype, stride, shape, region):
    # test_tensor.cpp:73-120 (serial oracle, region composition, stride-2 row map)
    rng = np.random.default_rng(sum(shape) + stride)
    x = rng.standard_normal(shape).astype(np.float32)
    w = (rng.standard_normal((7, shape[1], 3, 3)) / (3 * np.sqrt(shape[1]))).astype(np.float32)
    b = rng.standard_normal(7).astype(np.float32)
    got = conv(dtype, x, region, w, b, stride)
    ref = O.conv2d_region(x, region, w, b, stride, 1)
    assert got.shape == ref.shape
    assert O.rel_l2(got, ref) <= TOL[dtype], O.rel_l2(got, ref)


def test_conv_region_partitions_compose():
    # test_tensor.cpp:309-342: bands of a 12-row map reassemble the full conv
    rng = np.random.default_rng(3)
    x = rng.standard_normal((1, 8, 12, 8)).astype(np.float32)
    w = (rng.standard_normal((4, 8, 3, 3)) / 8).astype(np.float32)
    b = rng.standard_normal(4).astype(np.float32)
    full = conv("fp32", x, (0, 12), w, b, 1)
    for parts in (2, 3):
        band = 12 // parts
        pieces = [conv("fp32", x, (i * band, (i + 1) * band), w, b, 1) for i in range(parts)]
        assert np.array_equal(np.concatenate(pieces, axis=2), full)
    assert conv("fp32", x, (4, 8), w, b, 2).shape[2] == 2      # stride-2 row map [4,8) -> [2,4)


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
def test_linear_vs_oracle(dtype):
    rng = np.random.default_rng(5)
    t = rng.standard_normal((2, 1, 37, 48)).astype(np.float32)
    w = (rng.standard_normal((40, 48, 1, 1)) / 7).astype(np.float32)
    b = rng.standard_normal(40).astype(np.float32)
    out = np.zeros((2, 1, 37, 40), np.float32)
    N.check(N.lib().pp_linear(N.DTYPES[dtype], _p(t), 2, 37, 48, _p(w), 40, _p(b), _p(out)))
    assert O.rel_l2(out, O.linear(t, w, b)) <= TOL[dtype]


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
@pytest.mark.parametrize("m,s,d", [(1, 1, 8), (6, 10, 8), (128, 256, 64), (64, 1024, 1280),
                                   (200, 1000, 96), (128, 14400, 1280)])
def test_attention_vs_oracle(dtype, m, s, d):
    # test_tensor.cpp:148-175 (single token, oracle); d=1280 is the SDXL-shape head
    rng = np.random.default_rng(m + s + d)
    q = rng.standard_normal((1, 1, m, d)).astype(np.float32)
    k = rng.standard_normal((1, 1, s, d)).astype(np.float32)
    v = rng.standard_normal((1, 1, s, d)).astype(np.float32)
    scale = float(np.float32(1.0 / np.sqrt(d)))
    out = np.zeros((1, 1, m, d), np.float32)
    N.check(N.lib().pp_attention(N.DTYPES[dtype], _p(q), _p(k), _p(v), 1, m, s, d, d, scale, _p(out)))
    ref = O.attention(q, k, v, scale)
    assert O.rel_l2(out, ref) <= TOL[dtype] * 2, O.rel_l2(out, ref)
    if s == 1:
        assert np.allclose(out, np.broadcast_to(v[:, :, :1], out.shape), rtol=1e-2)


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
def test_attention_extreme_logit_ranges(dtype):
    # The softmax runs in the S-GEMM epilogue against each key tile's own row max; attn_rescale
    # brings the tiles to the row max.  One huge key puts the rows aligned with it ~50 above
    # every other logit (one tile dominates, the others are scaled by ~e^-50) while the
    # orthogonal rows see only O(1) logits: both must match the fp64 oracle.
    rng = np.random.default_rng(5)
    m, s, d = 64, 256, 64
    k = rng.standard_normal((1, 1, s, d)).astype(np.float32)
    k[0, 0, 3] = 0.0
    k[0, 0, 3, 0] = 400.0
    q = rng.standard_normal((1, 1, m, d)).astype(np.float32)
    q[0, 0, ::2, 0] = 0.0                      # orthogonal to the big key
    q[0, 0, 1::2] *= 0.05
    q[0, 0, 1::2, 0] = 1.0                     # aligned with it: one dominant logit
    v = rng.standard_normal((1, 1, s, d)).astype(np.float32)
    scale = float(np.float32(1.0 / np.sqrt(d)))
    out = np.zeros((1, 1, m, d), np.float32)
    N.check(N.lib().pp_attention(N.DTYPES[dtype], _p(q), _p(k), _p(v), 1, m, s, d, d, scale, _p(out)))
    ref = O.attention(q, k, v, scale)
    assert np.isfinite(out).all()
    for rows in (slice(0, None, 2), slice(1, None, 2)):
        err = O.rel_l2(out[0, 0, rows], ref[0, 0, rows])
        assert err <= TOL[dtype] * 2, (rows, err)


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
def test_group_stats_and_apply(dtype):
    # test_tensor.cpp:177-254: known stats, normalisation, oracle agreement, negative variance
    x = np.arange(16, dtype=np.float32).reshape(1, 16, 1, 1) * np.ones((1, 1, 2, 2), np.float32)
    mean = np.zeros(4)
    msq = np.zeros(4)
    N.check(N.lib().pp_group_stats(N.DTYPES[dtype], _p(f32(x)), 1, 16, 2, 2, 4, -1, -1, _p(mean), _p(msq)))
    assert np.allclose(mean, [1.5, 5.5, 9.5, 13.5])
    assert np.allclose(msq, [3.5, 31.5, 91.5, 183.5])
    rng = np.random.default_rng(9)
    x = (rng.standard_normal((1, 32, 8, 12)) * 2 + 0.5).astype(np.float32)
    om, oq = O.group_stats(x, 4, (2, 6))
    gm, gq = np.zeros(4), np.zeros(4)
    N.check(N.lib().pp_group_stats(N.DTYPES[dtype], _p(x), 1, 32, 8, 12, 4, 2, 6, _p(gm), _p(gq)))
    assert np.allclose(gm, om, rtol=1e-2, atol=1e-2) and np.allclose(gq, oq, rtol=1e-2)
    gamma = (1 + 0.1 * rng.standard_normal(32)).astype(np.float32)
    beta = (0.1 * rng.standard_normal(32)).astype(np.float32)
    out = np.zeros_like(x)
    N.check(N.lib().pp_group_norm_apply(N.DTYPES[dtype], _p(x), 1, 32, 8, 12, 2, 6, 4, _p(om), _p(oq),
                                        _p(gamma), _p(beta), 1e-5, _p(out)))
    ref = O.group_norm_apply(x, (2, 6), om, oq, gamma, beta, 1e-5)
    assert O.rel_l2(out, ref) <= TOL[dtype]
    assert np.array_equal(out[:, :, :2], x[:, :, :2])      # rows outside the region pass through
    bad_m, bad_q = np.array([1.0, 0, 0, 0]), np.array([0.5, 1, 1, 1])
    rc = N.lib().pp_group_norm_apply(N.DTYPES[dtype], _p(x), 1, 32, 8, 12, -1, -1, 4, _p(bad_m),
                                     _p(bad_q), _p(gamma), _p(beta), 1e-5, _p(out))
    assert rc == N.PP_ERUNTIME and "negative variance" in N.last_error()


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
def test_silu_upsample_ddim(dtype):
    rng = np.random.default_rng(11)
    x = (rng.standard_normal(1001) * 4).astype(np.float32)
    out = np.zeros_like(x)
    N.check(N.lib().pp_silu(N.DTYPES[dtype], _p(x), x.size, _p(out)))
    assert O.rel_l2(out, O.silu(x)) <= TOL[dtype]
    u = rng.standard_normal((1, 8, 3, 5)).astype(np.float32)
    uo = np.zeros((1, 8, 6, 10), np.float32)
    N.check(N.lib().pp_upsample_nearest2x(N.DTYPES[dtype], _p(u), 1, 8, 3, 5, _p(uo)))
    ref = O.upsample_nearest2x(u)
    assert np.array_equal(uo, ref) if dtype == "fp32" else O.rel_l2(uo, ref) <= 1e-2
    # DDIM closed form (test_sampler.cpp:66-73) -- the sampler is always fp32 / fp64
    one = np.ones(1, np.float32)
    y = np.zeros(1, np.float32)
    N.check(N.lib().pp_ddim_update(_p(one), _p(np.full(1, 0.5, np.float32)), 1, 0.25, 0.81, _p(y)))
    assert abs(float(y[0]) - 1.238522083771039) <= 1e-6
    xs = O.random_normal(1, 4, 16, 16, 3)
    es = O.random_normal(1, 4, 16, 16, 4)
    ys = np.zeros_like(xs)
    N.check(N.lib().pp_ddim_update(_p(xs), _p(es), xs.size, 0.3, 0.7, _p(ys)))
    assert np.array_equal(ys, O.ddim_update(xs, es, 0.3, 0.7))   # bit-exact fp64 math

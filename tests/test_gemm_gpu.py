"""tcgen05 GEMM / implicit-GEMM conv kernel vs a plain torch fp32/fp64 reference."""
import ctypes as C
import os

import pytest

torch = pytest.importorskip("torch")

from paper_2402_19481_b200 import _native as N  # noqa: E402

pytestmark = pytest.mark.gpu

# force_splits flag bits: run the CTA-pair (cta_group::2, M=256) or the single-CTA kernel
PAIR, SINGLE = 16, 32


def _p(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def _tf32(x):
    # round-to-nearest(away) to a 10-bit mantissa, like cvt.rna.tf32.f32
    i = x.contiguous().view(torch.int32)
    i = (i + 0x1000) & ~0x1FFF
    return i.view(torch.float32)


def gemm(dtype, A, B, bias=None, splits=0, bn=0, out_f32=True):
    M, K = A.shape
    Nn = B.shape[0]
    D = torch.zeros(M, Nn, device="cuda", dtype=torch.float32 if out_f32 else A.dtype)
    N.check(N.lib().pp_dev_gemm(N.DTYPES[dtype], _p(A), M, K, A.stride(0), _p(B), Nn, B.stride(0),
                                _p(bias), _p(D), D.stride(0), int(out_f32), splits, bn, None))
    return D


@pytest.mark.parametrize("M,Nn,K", [(128, 128, 64), (256, 320, 2880), (1000, 640, 576),
                                    (64, 16, 128), (1024, 1024, 1280), (128, 1280, 1024)])
@pytest.mark.parametrize("splits", [0, 1, 3])
@pytest.mark.parametrize("cta", [0, PAIR, SINGLE])
def test_gemm_bf16(M, Nn, K, splits, cta):
    g = torch.Generator(device="cuda").manual_seed(M + Nn + K)
    A = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    B = torch.randn(Nn, K, device="cuda", generator=g).bfloat16()
    bias = torch.randn(Nn, device="cuda", generator=g)
    D = gemm("bf16", A, B, bias, splits=splits | cta)
    ref = A.double() @ B.double().T + bias.double()
    err = (D.double() - ref).norm() / ref.norm()
    assert err < 1e-5, err


@pytest.mark.parametrize("M,Nn,K", [(128, 128, 32), (300, 320, 288), (1024, 1024, 1280)])
@pytest.mark.parametrize("cta", [0, PAIR, SINGLE])
def test_gemm_tf32(M, Nn, K, cta):
    g = torch.Generator(device="cuda").manual_seed(7)
    A = _tf32(torch.randn(M, K, device="cuda", generator=g))
    B = _tf32(torch.randn(Nn, K, device="cuda", generator=g))
    D = gemm("fp32", A, B, splits=cta)
    ref = A.double() @ B.double().T
    err = (D.double() - ref).norm() / ref.norm()
    assert err < 1e-5, err


def conv_ref(inp_pad, w, bias, stride):
    # inp_pad: [rows+2][W][C] (halo rows included); w: [co][3][3][C]
    x = inp_pad.double().permute(2, 0, 1).unsqueeze(0)
    wt = w.double().permute(0, 3, 1, 2)
    if stride == 2:
        x = x[:, :, :-1]
    y = torch.nn.functional.conv2d(x, wt, bias.double(), stride=stride, padding=(0, 1))
    return y[0].permute(1, 2, 0)  # [out_rows][out_w][co]


@pytest.mark.parametrize("rows,W,C,co,stride", [
    (4, 128, 64, 128, 1), (8, 64, 128, 320, 1), (16, 32, 64, 160, 1), (3, 120, 64, 64, 1),
    (5, 60, 64, 64, 1), (2, 240, 128, 64, 1), (8, 128, 64, 128, 2), (6, 64, 64, 64, 2),
    (4, 32, 320, 320, 1), (2, 16, 64, 16, 1)])
@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
def test_conv(rows, W, C, co, stride, dtype):
    g = torch.Generator(device="cuda").manual_seed(rows * 1000 + W + C)
    if dtype == "fp32" and C % 32:
        pytest.skip()
    inp = torch.randn(rows + 2, W, C, device="cuda", generator=g)
    w = torch.randn(co, 3, 3, C, device="cuda", generator=g) / (3 * C ** 0.5)
    bias = torch.randn(co, device="cuda", generator=g)
    if dtype == "bf16":
        inp, w = inp.bfloat16(), w.bfloat16()
    else:
        inp, w = _tf32(inp), _tf32(w)
    n_pad = (co + 15) // 16 * 16
    wp = torch.zeros(n_pad, 3, 3, C, device="cuda", dtype=w.dtype)
    wp[:co] = w
    orow = rows if stride == 1 else rows // 2
    ow = W if stride == 1 else W // 2
    out = torch.zeros(orow, ow, co, device="cuda", dtype=torch.float32)
    for splits in (0, 2, PAIR, PAIR | 2, SINGLE, SINGLE | 2):
        out.zero_()
        N.check(N.lib().pp_dev_conv(N.DTYPES[dtype], _p(inp), rows, W, C, stride, _p(wp), n_pad, co,
                                    _p(bias), _p(out), co, 1, None, 0, splits, 0, None))
        ref = conv_ref(inp, w, bias, stride)
        err = (out.double() - ref).norm() / ref.norm()
        assert err < 1e-5, (splits, err)


def test_conv_residual_bf16():
    g = torch.Generator(device="cuda").manual_seed(3)
    rows, W, C, co = 4, 64, 64, 64
    inp = torch.randn(rows + 2, W, C, device="cuda", generator=g).bfloat16()
    w = (torch.randn(co, 3, 3, C, device="cuda", generator=g) / 24).bfloat16()
    bias = torch.randn(co, device="cuda", generator=g)
    res = torch.randn(rows, W, co, device="cuda", generator=g).bfloat16()
    out = torch.zeros(rows, W, co, device="cuda", dtype=torch.bfloat16)
    N.check(N.lib().pp_dev_conv(0, _p(inp), rows, W, C, 1, _p(w), co, co, _p(bias), _p(out), co, 0,
                                _p(res), co, 0, 0, None))
    ref = conv_ref(inp, w, bias, 1) + res.double()
    err = (out.double() - ref).norm() / ref.norm()
    assert err < 1e-2, err

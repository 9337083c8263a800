"""Pins the torch fp64 restatement (oracle/patchsim_torch.py) to the numpy oracle.

The torch module re-executes the numpy oracle's source with torch float64 kernels; here it
runs on the CPU device against the numpy oracle in every run mode (toy model) and on the
SDXL-shape graph.  On the GPU box tests/test_parity_gpu.py also pins it to the reference
build (oracle/_ref) at the benchmarked 128x128 geometry.
"""
import numpy as np
import pytest

from oracle import patchsim_np as O
from oracle import patchsim_torch as PT


@pytest.fixture(scope="module")
def T():
    return PT.load("cpu")


@pytest.mark.parametrize("mode,n,warmup,scheme", [
    ("reference", 1, 4, "corrected"), ("sync-pp", 2, 4, "corrected"),
    ("displaced", 4, 0, "corrected"), ("displaced", 8, 1, "corrected"),
    ("displaced", 2, 0, "stale"), ("displaced", 4, 1, "separate"), ("naive", 2, 4, "corrected")])
def test_torch64_equals_numpy_oracle(T, mode, n, warmup, scheme):
    a = O.run_sampling(O.ModelConfig(), mode, n, 32, 32, 4, warmup, gn_scheme=scheme)
    b = T.run_sampling(T.ModelConfig(), mode, n, 32, 32, 4, warmup, gn_scheme=scheme)
    assert b["total_macs"] == a["total_macs"]
    for xa, xb in zip(a["trajectory"], b["trajectory"]):
        assert O.rel_l2(xb, xa) <= 1e-6
    assert O.rel_l2(b["x0"], a["x0"]) <= 1e-6


def test_torch64_sdxl_shape_forward(T):
    cfg = (4, 320, 3, 32, 2048, -1)
    om = O.build_model(O.ModelConfig(*cfg), 42)
    tm = T.build_model(T.ModelConfig(*cfg), 42)
    cond = O.random_condition(2048, 7)
    x = O.random_normal(1, 4, 32, 32, 1234)
    a = O.forward_full(om, x, 980, cond)
    b = T.to_host(T.forward_full(tm, x, 980, cond))
    assert O.rel_l2(b, a) <= 1e-6


def test_torch64_errors_match(T):
    r = T.PatchRunner(T.build_model(T.ModelConfig(), 1), O.random_condition(8, 2), 32, 32,
                      "displaced", 2, 0)
    with pytest.raises(T.RuntimeFailure, match="no cached activation for layer 0"):
        r.step_displaced(O.random_normal(1, 4, 32, 32, 3), 500, 1)
    x = O.random_normal(1, 4, 32, 32, 3)
    x[0, 0, 0, 0] = np.nan
    with pytest.raises(T.RuntimeFailure, match="non-finite"):
        T.PatchRunner(T.build_model(T.ModelConfig(), 1), O.random_condition(8, 2), 32, 32,
                      "reference").run_step(x, 500, 0)

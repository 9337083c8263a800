"""Host-side logic of the B200 runtime, through the C ABI, on CPU (no GPU needed).

Integer / index logic must match the reference bit-exactly: partitioning, patch specs
and their error texts, the weight pool (splitmix64 init), schedule / plan, Box-Muller
latents, MAC accounting, corrected GroupNorm statistics and RunConfig validation.
"""
import hashlib
import os

import numpy as np
import pytest

from oracle import patchsim_np as O
from paper_2402_19481_b200 import patchsim as P

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = np.load(os.path.join(HERE, "golden", "reference_golden.npz"), allow_pickle=True)
TINY = P.ModelConfig(2, 8, 2, 4, 8, -1)


def ocfg(c):
    return O.ModelConfig(c.in_channels, c.base_channels, c.levels, c.groups, c.cond_dim,
                         c.attn_at_level, c.res_blocks, c.attn_levels, c.attn_depth, c.attn_up)


DEEP = P.ModelConfig(4, 16, 3, 4, 8, -1, res_blocks=2, attn_levels=0b110, attn_depth=2, attn_up=1)


@pytest.mark.parametrize("cfg,seed", [(P.ModelConfig(), 42), (TINY, 77), (P.ModelConfig(3, 24, 4, 6, 5, 1), 9),
                                      (DEEP, 3)])
def test_weight_pool_bit_exact(cfg, seed):
    m = P.build_model(cfg, seed)
    om = O.build_model(ocfg(cfg), seed)
    ws = m.weights()
    assert len(ws) == len(om.weights)
    for a, b in zip(ws, om.weights):
        assert a.shape == b.shape and np.array_equal(a, b)
    for d, od in zip(m.layers, om.layers):
        assert d["kind"] == od.kind and d["skip_source"] == od.skip_source
        assert (d["in_ch"], d["out_ch"], d["stride"], d["scale_in"], d["scale_out"]) == \
               (od.in_ch, od.out_ch, od.stride, od.scale_in, od.scale_out)
        assert (d["weight"], d["bias"], d["weight2"], d["bias2"]) == \
               (od.weight, od.bias, od.weight2, od.bias2)


def test_sdxl_shape_pool_matches_reference_digest():
    m = P.build_model(P.SDXL_SHAPE, 42)
    pool = np.concatenate([w.reshape(-1) for w in m.weights()])
    assert pool.size == 77_388_804
    assert hashlib.sha256(pool.tobytes()).hexdigest() == str(GOLD["sdxl_weight_sha256"])
    assert m.total_macs(128, 128) == 231_234_600_960   # 0.2312 TMAC/step


def test_deeper_graph_topology():
    # beyond the reference API: the default extension fields build the reference graph (the
    # SDXL digest above); res_blocks / attn_levels / attn_depth / attn_up grow it -- level l
    # gets res_blocks residual blocks, each followed by attn_depth attention blocks at the
    # attention levels (and on the up path with attn_up)
    kinds = [d["kind"] for d in P.build_model(DEEP, 3).layers]
    base = [d["kind"] for d in P.build_model(P.ModelConfig(), 3).layers]
    assert kinds.count("SelfAttn") == 2 * 2 * 2 + 2 * 2 * 1   # down: 2 lv x 2 rb x 2; up: lv 1 only
    assert kinds.count("Conv") == base.count("Conv") + 4 * 2 + 2 * 2 - 2
    assert base.count("SelfAttn") == 1
    for bad in (dict(res_blocks=-1), dict(attn_depth=-2), dict(attn_levels=8)):
        with pytest.raises(P.InvalidArgument, match="ModelConfig"):
            P.build_model(P.ModelConfig(**bad), 1)


def test_from_pool_roundtrip():
    m = P.build_model(P.ModelConfig(), 5)
    ws = m.weights()
    m2 = P.Model.from_pool(P.ModelConfig(), ws)
    assert all(np.array_equal(a, b) for a, b in zip(ws, m2.weights()))
    with pytest.raises(P.InvalidArgument, match="weight pool"):
        P.Model.from_pool(P.ModelConfig(), ws[:-1])


def test_partition_rows():
    # proj/tests/test_runtime.cpp:49-61
    assert P.partition_rows(8, 2, 8) == [(0, 4, 8, 8), (4, 8, 8, 8)]
    assert P.partition_rows(8, 1, 8) == [(0, 8, 8, 8)]
    with pytest.raises(P.InvalidArgument, match="not divisible by 3 devices"):
        P.partition_rows(8, 3, 8)


def test_patch_specs_bit_exact_against_reference():
    for row in GOLD["patch_specs"]:
        cfg = P.ModelConfig(*[int(v) for v in row[:6]])
        reg = tuple(int(v) for v in row[9:13])
        m = P.build_model(cfg, 1)
        lin, lout = m.patch_spec(reg)
        L = lin.shape[0]
        got = np.concatenate([lin.reshape(-1), lout.reshape(-1)])
        assert np.array_equal(got, np.array(row[13:13 + 8 * L], dtype=np.int64))


def test_patch_spec_divisibility_error_text():
    # proj/tests/test_runtime.cpp:63-72
    m = P.build_model(P.ModelConfig(), 1)
    with pytest.raises(P.InvalidArgument, match="not divisible at layer 20 \\(DownConv\\)"):
        m.patch_spec(P.partition_rows(48, 8, 48)[1])
    for r in P.partition_rows(48, 4, 48):
        m.patch_spec(r)


def test_corrected_gn_stats_cases():
    # proj/tests/test_runtime.cpp:188-229, through the C ABI
    fresh = ([0.5, 1.0], [0.5, 2.0])
    pl = ([0.4, 0.9], [0.45, 1.8])
    pg = ([0.42, 0.95], [0.48, 1.9])
    for args in [(pl, pl, pg), (fresh, pl, pl), (fresh, pl, pg),
                 (([0.0], [0.085]), ([0.0], [0.1]), ([1.0], [1.005]))]:
        a = P.corrected_gn_stats(*args)
        b = O.corrected_gn_stats(*args)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    with pytest.raises(P.InvalidArgument):
        P.corrected_gn_stats(fresh, pl, ([0.1, 0.2, 0.3], [0.1, 0.2, 0.3]))


def test_schedule_plan_and_rng():
    assert np.array_equal(P.make_schedule(), GOLD["abar"])
    assert P.make_plan(1000, 50) == list(GOLD["plan50"])
    assert P.make_plan(1000, 4) == [750, 500, 250, 0]
    with pytest.raises(P.InvalidArgument):
        P.make_plan(1000, 0)
    assert np.array_equal(P.random_normal(1, 4, 32, 32, 1234), O.random_normal(1, 4, 32, 32, 1234))
    assert np.array_equal(P.random_condition(2048, 7), O.random_condition(2048, 7))
    assert np.array_equal(P.random_normal(1, 1, 1, 3, 5), O.random_normal(1, 1, 1, 3, 5))


def test_macs_of_layer_and_totals():
    m = P.build_model(P.SDXL_SHAPE, 1)
    om = O.build_model(O.SDXL_SHAPE, 1, fill=False)
    for lat in (32, 128, 256, 480):
        assert m.total_macs(lat, lat) == O.model_total_macs(om, lat, lat)
    for reg in P.partition_rows(128, 8, 128):
        lin, _ = m.patch_spec(reg)
        for d, r in zip(om.layers, lin):
            reg4 = tuple(int(v) for v in r)
            assert m.macs_of_layer(d.id, reg4) == O.macs_of_layer(d, reg4)


def test_run_config_validate():
    P.RunConfig(mode="displaced", n_devices=2, h=32, w=32, num_steps=4).validate()
    with pytest.raises(P.InvalidArgument, match="devices\\*2\\^\\(levels-1\\)"):
        P.RunConfig(mode="sync-pp", n_devices=3, h=16, w=16, model=TINY, num_steps=2).validate()
    with pytest.raises(P.InvalidArgument, match="must be divisible"):
        P.RunConfig(mode="displaced", n_devices=8, h=160, w=240, model=P.SDXL_SHAPE).validate()
    with pytest.raises(P.InvalidArgument, match="steps out of range"):
        P.RunConfig(num_steps=0).validate()
    with pytest.raises(P.InvalidArgument, match="warmup"):
        P.RunConfig(warmup=-1).validate()


def test_runner_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    m = P.build_model(P.ModelConfig(), 1)
    with pytest.raises(P.CudaError, match="no CPU fallback"):
        P.PatchRunner(m, np.zeros(8, np.float32), 16, 16)

"""Pin the CPU oracle (oracle/patchsim_np.py) before trusting it.

Checks against (1) the golden vectors held by the reference's own tests, (2) the
committed fixtures generated from the reference build (tests/golden/make_golden.py),
and (3) the reference itself (oracle/_ref) when it can be built here.
"""
import hashlib
import os

import numpy as np
import pytest

from oracle import patchsim_np as O

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = np.load(os.path.join(HERE, "golden", "reference_golden.npz"), allow_pickle=True)


def fnv(a):
    from oracle.ref import fnv1a64
    return fnv1a64(a)


def test_golden_forward_hash():
    # proj/tests/test_model.cpp:234-246
    m = O.build_model(O.TOY, 42)
    y = O.forward_full(m, np.zeros((1, 4, 16, 16), np.float32), 10, np.zeros(8, np.float32))
    assert fnv(y) == 0x67EC5910FD4BB9F3
    assert np.array_equal(y, GOLD["golden_forward"])


def test_model_graph_counts():
    # proj/tests/test_model.cpp:201-214
    m = O.build_model(O.TOY, 42)
    assert len(m.layers) == 63
    assert sum(d.needs_gather() for d in m.layers) == 17
    assert sum(d.kind == "GroupNorm" for d in m.layers) == 11
    sd = O.build_model(O.SDXL_SHAPE, 42)
    assert sum(w.size for w in sd.weights) == 77_388_804
    digest = hashlib.sha256(np.concatenate([w.reshape(-1) for w in sd.weights]).tobytes()).hexdigest()
    assert digest == str(GOLD["sdxl_weight_sha256"])


def test_forward_collect_matches_reference_layer_by_layer():
    m = O.build_model(O.TOY, 77)
    outs = O.forward_collect(m, GOLD["toy_collect_x"], 700, GOLD["toy_collect_cond"])
    for i, o in enumerate(outs):
        ref = GOLD[f"toy_collect_{i:02d}"]
        assert o.shape == ref.shape
        assert O.rel_l2(o, ref) <= 1e-6, i


def test_sdxl_shape_forward():
    m = O.build_model(O.SDXL_SHAPE, 42)
    cond = O.random_condition(2048, 7)
    assert np.array_equal(GOLD["sdxl16_x"], O.random_normal(1, 4, 16, 16, 1234))
    eps = O.forward_full(m, GOLD["sdxl16_x"], 980, cond)
    assert O.rel_l2(eps, GOLD["sdxl16_eps"]) <= 1e-6


@pytest.mark.parametrize("mode,n,wu,hexhash", [
    ("reference", 1, 4, 0xB855148A7BE1688C), ("displaced", 2, 1, 0x988768A7E072F109),
    ("displaced", 2, 0, 0x43B760DB1277531A), ("sync-pp", 2, 4, 0xB855148A7BE1688C),
    ("naive", 2, 4, None), ("displaced", 4, 1, None)])
def test_c1_run_sampling(mode, n, wu, hexhash):
    # BASELINE config 1; hashes from SURVEY.md §8c (measured on the reference build)
    r = O.run_sampling(O.TOY, mode, n, 32, 32, 4, wu)
    key = f"c1_{mode}_n{n}_w{wu}"
    assert np.array_equal(r["x0"], GOLD[key + "_x0"])
    for i, xt in enumerate(r["trajectory"]):
        assert np.array_equal(xt, GOLD[key + "_traj"][i])
    assert r["total_macs"] == int(GOLD[key + "_macs"][0])
    if hexhash is not None:
        assert fnv(r["x0"]) == hexhash


def test_sampler_closed_forms():
    # proj/tests/test_sampler.cpp:38-73
    assert O.make_plan(1000, 50) == list(GOLD["plan50"])
    assert O.make_plan(1000, 50)[0] == 980 and O.make_plan(1000, 50)[-1] == 0
    assert np.array_equal(O.make_schedule(), GOLD["abar"])
    y = O.ddim_update(np.ones((1, 1, 1, 1), np.float32), np.full((1, 1, 1, 1), 0.5, np.float32),
                      0.25, 0.81)
    assert abs(float(y[0, 0, 0, 0]) - 1.238522083771039) <= 1e-6
    x = O.random_normal(1, 1, 4, 4, 7)
    z = O.ddim_update(x, np.zeros_like(x), 0.25, 0.64)
    assert np.allclose(z, np.sqrt(0.64 / 0.25) * x, atol=1e-6)


def test_corrected_gn_stats_cases():
    # proj/tests/test_runtime.cpp:188-229
    fresh = ([0.5, 1.0], [0.5, 2.0])
    pl = ([0.4, 0.9], [0.45, 1.8])
    pg = ([0.42, 0.95], [0.48, 1.9])
    m, q = O.corrected_gn_stats(pl, pl, pg)
    assert list(m) == pg[0] and list(q) == pg[1]
    m, q = O.corrected_gn_stats(fresh, pl, pl)
    assert list(m) == fresh[0] and list(q) == fresh[1]
    m, q = O.corrected_gn_stats(fresh, pl, pg)
    assert m[0] == pytest.approx(0.42 + 0.1) and q[0] == pytest.approx(0.48 + 0.05)
    m, q = O.corrected_gn_stats(([0.0], [0.085]), ([0.0], [0.1]), ([1.0], [1.005]))
    assert m[0] == 0.0 and q[0] == 0.085
    with pytest.raises(O.InvalidArgument):
        O.corrected_gn_stats(fresh, pl, ([0.1, 0.2, 0.3], [0.1, 0.2, 0.3]))


def test_partition_and_patch_specs():
    # proj/tests/test_runtime.cpp:49-72 and the BASELINE geometries (bit-exact ints)
    assert O.partition_rows(8, 2, 8) == [(0, 4, 8, 8), (4, 8, 8, 8)]
    with pytest.raises(O.InvalidArgument):
        O.partition_rows(8, 3, 8)
    m = O.build_model(O.TOY, 1)
    with pytest.raises(O.InvalidArgument, match="not divisible"):
        O.derive_patch_spec(m, O.partition_rows(48, 8, 48)[1])
    for row in GOLD["patch_specs"]:
        cfg = O.ModelConfig(*[int(v) for v in row[:6]])
        h, w, n = (int(v) for v in row[6:9])
        reg = tuple(int(v) for v in row[9:13])
        mm = O.build_model(cfg, 1, fill=False)
        lin, lout = O.derive_patch_spec(mm, reg)
        L = len(mm.layers)
        got = np.concatenate([np.array(lin).reshape(-1), np.array(lout).reshape(-1)])
        assert np.array_equal(got, np.array(row[13:13 + 8 * L], dtype=np.int64))


def test_run_config_validate_rejects_config3():
    # 1280x1920 (160x240 latent) at N=8 fails RunConfig::validate
    with pytest.raises(O.InvalidArgument, match="must be divisible"):
        O.run_config_validate(O.SDXL_SHAPE, "displaced", 8, 160, 240, 50, 4)


ref_available = pytest.mark.skipif(
    not os.path.isdir("/root/reference/proj") and not os.path.exists(
        os.path.join(os.path.dirname(HERE), "oracle", "_ref", "libpatchsim_ref.so")),
    reason="reference build not available")


@ref_available
@pytest.mark.parametrize("mode,n,wu", [("sync-pp", 4, 4), ("displaced", 4, 0), ("naive", 4, 4)])
def test_oracle_vs_reference_build_48(mode, n, wu):
    from oracle import ref as R
    a = O.run_sampling(O.TOY, mode, n, 48, 48, 3, wu)
    b = R.run_sampling(O.TOY.as_tuple(), mode, n, 48, 48, 3, wu)
    assert np.array_equal(a["x0"], b["x0"])
    assert a["total_macs"] == b["total_macs"]


@ref_available
def test_oracle_kernels_vs_reference_build():
    from oracle import ref as R
    rng = np.random.default_rng(0)
    x = rng.standard_normal((1, 5, 9, 7)).astype(np.float32)
    w = rng.standard_normal((3, 5, 3, 3)).astype(np.float32)
    b = rng.standard_normal(3).astype(np.float32)
    for stride, reg in [(1, (0, 9)), (1, (3, 6)), (2, (2, 8)), (2, (0, 9))]:
        assert O.rel_l2(O.conv2d_region(x, reg, w, b, stride, 1),
                        R.conv2d_region(x, reg, w, b, stride, 1)) <= 1e-7
    q = rng.standard_normal((1, 1, 6, 8)).astype(np.float32)
    k = rng.standard_normal((1, 1, 10, 8)).astype(np.float32)
    v = rng.standard_normal((1, 1, 10, 4)).astype(np.float32)
    assert O.rel_l2(O.attention(q, k, v, 0.3), R.attention(q, k, v, 0.3)) <= 1e-7
    g = rng.standard_normal((1, 8, 4, 4)).astype(np.float32)
    m1, q1 = O.group_stats(g, 4)
    m2, q2 = R.group_stats(g, 4)
    assert np.allclose(m1, m2, rtol=1e-12) and np.allclose(q1, q2, rtol=1e-12)

"""B200 PatchRunner / run_sampling parity against the CPU oracle (numpy restatement,
pinned to the reference in tests/test_oracle.py).

Tolerances (BASELINE.json north_star): relative L2 <= 1e-3 in fp32-accumulate mode
(fp32 storage, TF32 tensor cores) and <= 2e-2 in bf16.  Patch partitioning and halo
indexing are integer logic and are compared bit-exactly elsewhere.
"""
import dataclasses

import numpy as np
import pytest

from oracle import patchsim_np as O
from paper_2402_19481_b200 import patchsim as P

pytestmark = pytest.mark.gpu

TOL = {"fp32": 1e-3, "bf16": 2e-2}          # per-step latents x_t (north-star bar)
# A single eps evaluation is not damped by the sampler; 63 layers of TF32 / bf16
# rounding give ~1e-3 / ~1e-2 relative error on eps itself.
EPS_TOL = {"fp32": 3e-3, "bf16": 3e-2}
TINY = P.ModelConfig(2, 8, 2, 4, 8, -1)        # proj/tests/test_runtime.cpp:16-24
TOY = P.ModelConfig()                           # model.hpp:30-36 defaults


def ocfg(c):
    return O.ModelConfig(c.in_channels, c.base_channels, c.levels, c.groups, c.cond_dim,
                         c.attn_at_level, c.res_blocks, c.attn_levels, c.attn_depth, c.attn_up)


def rel(a, b):
    return O.rel_l2(a, b)


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
@pytest.mark.parametrize("cfg,hw", [(TOY, 32), (TINY, 16)])
def test_reference_forward(dtype, cfg, hw):
    om = O.build_model(ocfg(cfg), 77)
    cond = O.random_condition(cfg.cond_dim, 78)
    x = O.random_normal(1, cfg.in_channels, hw, hw, 79)
    ref = O.forward_full(om, x, 700, cond)
    m = P.build_model(cfg, 77)
    r = P.PatchRunner(m, cond, hw, hw, mode="reference", dtype=dtype)
    eps = r.run_step(x, 700, 0)
    assert rel(eps, ref) <= EPS_TOL[dtype], rel(eps, ref)


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
@pytest.mark.parametrize("n", [2, 4])
def test_sync_matches_reference(dtype, n):
    # proj/tests/test_runtime.cpp:231-248 (sync-pp == reference forward)
    cfg, hw = TOY, 32
    om = O.build_model(ocfg(cfg), 77)
    cond = O.random_condition(cfg.cond_dim, 78)
    x = O.random_normal(1, cfg.in_channels, hw, hw, 79)
    ref = O.forward_full(om, x, 700, cond)
    r = P.PatchRunner(P.build_model(cfg, 77), cond, hw, hw, mode="sync-pp", n_devices=n,
                      dtype=dtype)
    eps = r.step_sync(x, 700, 0)
    assert rel(eps, ref) <= EPS_TOL[dtype], rel(eps, ref)


@pytest.mark.parametrize("n", [1, 2, 4])
def test_zero_staleness_displaced_equals_sync(n):
    # proj/tests/test_runtime.cpp:263-280
    cfg, hw = TOY, 32
    cond = O.random_condition(cfg.cond_dim, 88)
    x = O.random_normal(1, cfg.in_channels, hw, hw, 89)
    m = P.build_model(cfg, 87)
    d = P.PatchRunner(m, cond, hw, hw, mode="displaced", n_devices=n, dtype="fp32")
    d.step_sync(x, 700, 0)
    e_disp = d.step_displaced(x, 700, 1)
    s = P.PatchRunner(m, cond, hw, hw, mode="sync-pp", n_devices=n, dtype="fp32")
    e_sync = s.step_sync(x, 700, 0)
    assert rel(e_disp, e_sync) <= 1e-5


def test_missing_cache_names_the_layer():
    # proj/tests/test_runtime.cpp:282-290
    m = P.build_model(TINY, 97)
    cond = O.random_condition(8, 98)
    r = P.PatchRunner(m, cond, 16, 16, mode="displaced", n_devices=2, dtype="bf16")
    x = O.random_normal(1, 2, 16, 16, 99)
    with pytest.raises(P.RuntimeFailure, match="no cached activation for layer"):
        r.step_displaced(x, 500, 1)


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
@pytest.mark.parametrize("mode,n,warmup", [("reference", 1, 4), ("sync-pp", 2, 4),
                                           ("displaced", 2, 0), ("displaced", 2, 1),
                                           ("displaced", 4, 1)])
def test_run_sampling_c1(dtype, mode, n, warmup):
    # BASELINE config 1: toy model, 32x32 latent, 4 steps, 2 patches; trajectory per step
    cfg = TOY
    ref = O.run_sampling(ocfg(cfg), mode, n, 32, 32, 4, warmup)
    got = P.run_sampling(P.RunConfig(mode=mode, n_devices=n, h=32, w=32, num_steps=4,
                                     warmup=warmup, dtype=dtype, model=cfg), trajectory=True)
    for i, xt in enumerate(ref["trajectory"]):
        assert rel(got["trajectory"][i], xt) <= TOL[dtype], (i, rel(got["trajectory"][i], xt))
    assert rel(got["x0"], ref["x0"]) <= TOL[dtype], rel(got["x0"], ref["x0"])
    assert got["total_macs"] == ref["total_macs"]


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
@pytest.mark.parametrize("mode,n", [("reference", 1), ("displaced", 2)])
def test_sdxl_shape_small(dtype, mode, n):
    # SDXL-shape graph (320/640/1280 ch, GN32, d=1280 attention) on a 32x32 latent, 3 steps
    cfg = P.SDXL_SHAPE
    ref = O.run_sampling(ocfg(cfg), mode, n, 32, 32, 3, 0)
    got = P.run_sampling(P.RunConfig(mode=mode, n_devices=n, h=32, w=32, num_steps=3, warmup=0,
                                     dtype=dtype, model=cfg), trajectory=True)
    for i, xt in enumerate(ref["trajectory"]):
        assert rel(got["trajectory"][i], xt) <= TOL[dtype], (i, rel(got["trajectory"][i], xt))
    assert rel(got["x0"], ref["x0"]) <= TOL[dtype], rel(got["x0"], ref["x0"])


@pytest.mark.parametrize("mode,n", [("displaced", 1), ("displaced", 2), ("sync-pp", 4)])
def test_graph_replay_is_bit_identical(mode, n):
    # The denoising loop is captured into a CUDA graph on the first sample() and replayed
    # afterwards; the eager path (trajectory=True disables the graph) must agree bitwise,
    # and so must repeated replays (no float atomics anywhere: run-to-run determinism).
    cfg = TOY
    m = P.build_model(cfg, 42)
    cond = O.random_condition(cfg.cond_dim, 7)
    x = O.random_normal(1, cfg.in_channels, 32, 32, 1234)
    abar = O.make_schedule()
    plan = O.make_plan(1000, 6)
    r = P.PatchRunner(m, cond, 32, 32, mode=mode, n_devices=n, warmup_steps=1, dtype="bf16")
    eager, _ = r.sample(x, plan, abar, trajectory=True)
    g1, _ = r.sample(x, plan, abar)
    g2, _ = r.sample(x, plan, abar)
    assert np.array_equal(g1, eager)
    assert np.array_equal(g2, g1)
    ref = O.run_sampling(ocfg(cfg), mode, n, 32, 32, 6, 1)["x0"]
    assert rel(g2, ref) <= TOL["bf16"]


@pytest.mark.parametrize("mode,n", [("displaced", 4), ("sync-pp", 2)])
def test_stress_sched_does_not_change_results(mode, n):
    # --stress-sched (CollectiveHub::maybe_stress, collectives.cpp:45-56): seeded sleep kernels
    # on the compute and exchange streams around every exchange perturb the schedule; the
    # exchange is ordered by events, so x0 (eager and graph-replayed) is bitwise unchanged
    cfg = TOY
    m = P.build_model(cfg, 42)
    cond = O.random_condition(cfg.cond_dim, 7)
    x = O.random_normal(1, cfg.in_channels, 32, 32, 1234)
    abar = O.make_schedule()
    plan = O.make_plan(1000, 6)
    outs = []
    for stress, seed in ((False, 0xC0FFEE), (True, 0xC0FFEE), (True, 99)):
        r = P.PatchRunner(m, cond, 32, 32, mode=mode, n_devices=n, warmup_steps=1, dtype="bf16",
                          stress=stress, stress_seed=seed)
        eager, _ = r.sample(x, plan, abar, trajectory=True)
        g, _ = r.sample(x, plan, abar)
        outs += [eager, g]
    for o in outs[1:]:
        assert np.array_equal(o, outs[0])


def test_graph_replay_after_other_plan_uses_its_own_time_embeddings():
    # sample(A) captures the graph; an eager sample(B) (trajectory=True) rewrites the per-plan
    # time-embedding table in place; the next sample(A) replays the graph and must see A's
    # embeddings again (bitwise equal to an eager run of A)
    cfg = TOY
    m = P.build_model(cfg, 42)
    cond = O.random_condition(cfg.cond_dim, 7)
    x = O.random_normal(1, cfg.in_channels, 32, 32, 1234)
    abar = O.make_schedule()
    plan_a = O.make_plan(1000, 6)
    plan_b = [900, 700, 500, 300]     # shorter plan: fits the table in place
    r = P.PatchRunner(m, cond, 32, 32, mode="displaced", n_devices=2, warmup_steps=1,
                      dtype="bf16")
    eager_a, _ = r.sample(x, plan_a, abar, trajectory=True)
    g1, _ = r.sample(x, plan_a, abar)
    r.sample(x, plan_b, abar, trajectory=True)
    g2, _ = r.sample(x, plan_a, abar)
    assert np.array_equal(g1, eager_a)
    assert np.array_equal(g2, eager_a)


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
@pytest.mark.parametrize("n", [2, 4])
def test_run_sampling_naive(dtype, n):
    # ablation config 5 (naive patches): rows on even steps, columns on odd steps,
    # every patch an independent image (runtime.cpp:398-452)
    cfg = TOY
    ref = O.run_sampling(ocfg(cfg), "naive", n, 32, 32, 4, 4)
    got = P.run_sampling(P.RunConfig(mode="naive", n_devices=n, h=32, w=32, num_steps=4,
                                     warmup=4, dtype=dtype, model=cfg), trajectory=True)
    for i, xt in enumerate(ref["trajectory"]):
        assert rel(got["trajectory"][i], xt) <= TOL[dtype], (i, rel(got["trajectory"][i], xt))
    assert rel(got["x0"], ref["x0"]) <= TOL[dtype], rel(got["x0"], ref["x0"])
    assert got["total_macs"] == ref["total_macs"]


@pytest.mark.parametrize("step", [0, 1])
def test_naive_step_rows_and_columns(step):
    cfg, hw, n = TOY, 32, 2
    om = O.build_model(ocfg(cfg), 5)
    cond = O.random_condition(cfg.cond_dim, 6)
    x = O.random_normal(1, cfg.in_channels, hw, hw, 7)
    orr = O.PatchRunner(om, cond, hw, hw, mode="naive", n_devices=n)
    ref = orr.step_naive(x, 600, step)
    r = P.PatchRunner(P.build_model(cfg, 5), cond, hw, hw, mode="naive", n_devices=n, dtype="fp32")
    eps = r.step_naive(x, 600, step)
    assert rel(eps, ref) <= EPS_TOL["fp32"], rel(eps, ref)
    assert r.total_macs() == orr.total_macs
    assert r.step_device_macs(step) == orr.step_device_macs[step]


def test_naive_geometry_errors():
    m = P.build_model(TOY, 1)
    cond = O.random_condition(TOY.cond_dim, 2)
    x = O.random_normal(1, TOY.in_channels, 32, 32, 3)
    r = P.PatchRunner(m, cond, 32, 32, mode="naive", n_devices=3, dtype="bf16")
    with pytest.raises(P.InvalidArgument, match="naive: extent 32 not divisible by 3 devices"):
        r.step_naive(x, 500, 0)
    r = P.PatchRunner(m, cond, 32, 32, mode="naive", n_devices=16, dtype="bf16")
    with pytest.raises(P.InvalidArgument,
                       match=r"naive: patch extent 2 violates model divisibility \(4\)"):
        r.step_naive(x, 500, 0)


def test_naive_sample_is_deterministic():
    cfg = TOY
    m = P.build_model(cfg, 42)
    cond = O.random_condition(cfg.cond_dim, 7)
    x = O.random_normal(1, cfg.in_channels, 32, 32, 1234)
    abar = O.make_schedule()
    plan = O.make_plan(1000, 5)
    r = P.PatchRunner(m, cond, 32, 32, mode="naive", n_devices=2, dtype="bf16")
    a, _ = r.sample(x, plan, abar)
    b, _ = r.sample(x, plan, abar)
    assert np.array_equal(a, b)
    ref = O.run_sampling(ocfg(cfg), "naive", 2, 32, 32, 5, 4)["x0"]
    assert rel(a, ref) <= TOL["bf16"]


def _ref_lib():
    from oracle import ref as R
    if not R.available():
        pytest.skip("oracle/_ref (reference build) not available")
    return R


@pytest.mark.parametrize("mode,n,warmup", [("displaced", 2, 1), ("displaced", 4, 0), ("sync-pp", 2, 4),
                                           ("reference", 1, 4), ("naive", 2, 4), ("displaced", 1, 1)])
def test_trace_matches_reference(mode, n, warmup):
    # RawTrace (proj/include/patchsim/trace.hpp:18-35) of the B200 runner == the reference
    # PatchRunner's trace for the same run_step calls, event by event
    R = _ref_lib()
    cfg, hw = TOY, 32
    cond = O.random_condition(cfg.cond_dim, 7)
    x = O.random_normal(1, cfg.in_channels, hw, hw, 1234)
    rm = R.Model(dataclasses.astuple(cfg), 42)
    rr = R.PatchRunner(rm, cond, hw, hw, mode=mode, n_devices=n, warmup=warmup)
    pr = P.PatchRunner(P.build_model(cfg, 42), cond, hw, hw, mode=mode, n_devices=n,
                       warmup_steps=warmup, dtype="bf16")
    for s, t in enumerate([750, 500, 250, 0]):
        rr.step("run_step", x, t, s)
        pr.run_step(x, t, s)
    for d in range(pr.n_devices):
        assert pr.trace(d) == rr.trace(d), d


def test_trace_after_graph_sample_matches_reference():
    R = _ref_lib()
    cfg, hw = TOY, 32
    cond = O.random_condition(cfg.cond_dim, 7)
    x = O.random_normal(1, cfg.in_channels, hw, hw, 1234)
    abar = O.make_schedule()
    plan = O.make_plan(1000, 4)
    pr = P.PatchRunner(P.build_model(cfg, 42), cond, hw, hw, mode="displaced", n_devices=2,
                       warmup_steps=1, dtype="bf16")
    pr.sample(x, plan, abar)
    pr.sample(x, plan, abar)   # second call replays the captured CUDA graph
    # every sample() is a fresh run (run_sampling builds a new PatchRunner, runtime.cpp:494-526)
    expect = {0: [], 1: []}
    for _ in range(2):
        rr = R.PatchRunner(R.Model(dataclasses.astuple(cfg), 42), cond, hw, hw, mode="displaced",
                           n_devices=2, warmup=1)
        for s, t in enumerate(plan):
            rr.step("run_step", x, int(t), s)
        for d in range(2):
            expect[d] += rr.trace(d)
    for d in range(2):
        assert pr.trace(d) == expect[d], d


@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
def test_reference_forward_wide_latent(dtype):
    # a 128-pixel-wide latent puts the level-0 convs on the slab path (one im2col slab per
    # channel chunk serves all nine taps) and on CTA pairs; same parity bar as the toy sizes
    cfg, h, w = TOY, 64, 128
    om = O.build_model(ocfg(cfg), 17)
    cond = O.random_condition(cfg.cond_dim, 18)
    x = O.random_normal(1, cfg.in_channels, h, w, 19)
    ref = O.forward_full(om, x, 400, cond)
    r = P.PatchRunner(P.build_model(cfg, 17), cond, h, w, mode="reference", dtype=dtype)
    eps = r.run_step(x, 400, 0)
    assert rel(eps, ref) <= EPS_TOL[dtype], rel(eps, ref)


def test_displaced_wide_latent_matches_oracle():
    cfg, h, w = TOY, 64, 128
    res = O.run_sampling(ocfg(cfg), "displaced", 2, h, w, 4, 1)
    m = P.build_model(cfg, 42)
    cond = O.random_condition(cfg.cond_dim, 7)
    x = O.random_normal(1, cfg.in_channels, h, w, 1234)
    abar = O.make_schedule()
    plan = O.make_plan(1000, 4)
    r = P.PatchRunner(m, cond, h, w, mode="displaced", n_devices=2, warmup_steps=1, dtype="bf16")
    x0, _ = r.sample(x, plan, abar)
    assert rel(x0, res["x0"]) <= TOL["bf16"], rel(x0, res["x0"])


SDXL = P.ModelConfig(4, 320, 3, 32, 2048, -1)   # the SDXL-shape graph


@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
def test_sdxl_shape_forward_matches_reference_build(dtype):
    # the benchmark's model (320/640/1280 channels, GN32, d=1280 attention, 77.4M params) at a
    # 32x32 latent: one eps against the reference's own CPU path (oracle/_ref), same weights
    R = _ref_lib()
    hw = 32
    cond = O.random_condition(2048, 7)
    x = O.random_normal(1, 4, hw, hw, 1234)
    rr = R.PatchRunner(R.Model(dataclasses.astuple(SDXL), 42), cond, hw, hw, mode="reference")
    ref = rr.step("run_step", x, 980, 0)
    r = P.PatchRunner(P.build_model(SDXL, 42), cond, hw, hw, mode="reference", dtype=dtype)
    eps = r.run_step(x, 980, 0)
    assert rel(eps, ref) <= EPS_TOL[dtype], rel(eps, ref)


def test_sdxl_shape_displaced_two_bands_matches_reference_build():
    # displaced patch parallelism at the real channel counts: 2 bands, warm-up 1, 3 steps of
    # DDIM through run_step on both sides (halo rows, full K/V and GN statistics exchanged)
    R = _ref_lib()
    hw = 32
    cond = O.random_condition(2048, 7)
    x = O.random_normal(1, 4, hw, hw, 1234)
    abar = O.make_schedule()
    plan = [980, 960, 940]
    rr = R.PatchRunner(R.Model(dataclasses.astuple(SDXL), 42), cond, hw, hw, mode="displaced",
                       n_devices=2, warmup=1)
    pr = P.PatchRunner(P.build_model(SDXL, 42), cond, hw, hw, mode="displaced", n_devices=2,
                       warmup_steps=1, dtype="bf16")
    xr, xp = x.copy(), x.copy()
    for s, t in enumerate(plan):
        er = rr.step("run_step", xr, t, s)
        ep = pr.run_step(xp, t, s)
        assert rel(ep, er) <= EPS_TOL["bf16"], (s, rel(ep, er))
        tn = plan[s + 1] if s + 1 < len(plan) else -1
        a_t, a_n = O.alpha_bar_at(abar, t), O.alpha_bar_at(abar, tn)
        xr = O.ddim_update(xr, er, a_t, a_n)
        xp = O.ddim_update(xp, ep, a_t, a_n)
    assert rel(xp, xr) <= TOL["bf16"], rel(xp, xr)


@pytest.mark.parametrize("entry,mode,n", [("run_step", "reference", 1), ("run_step", "sync-pp", 2),
                                          ("step_naive", "naive", 2)])
def test_non_finite_input_is_reported(entry, mode, n):
    # Tensor::require_finite (proj/src/tensor.cpp:36-42) on the step's eps
    # (proj/src/runtime.cpp:346-394): runtime_error "<who>: non-finite value in tensor (1,C,H,W)"
    m = P.build_model(TINY, 97)
    cond = O.random_condition(8, 98)
    r = P.PatchRunner(m, cond, 16, 16, mode=mode, n_devices=n, dtype="bf16")
    x = O.random_normal(1, 2, 16, 16, 99)
    x[0, 1, 7, 3] = np.nan
    # run_step dispatches Reference mode to step_reference, which names itself (runtime.cpp:394)
    who = {"naive": "step_naive", "reference": "step_reference"}.get(mode, "run_step")
    with pytest.raises(P.RuntimeFailure, match=rf"{who}: non-finite value in tensor \(1,2,16,16\)"):
        getattr(r, entry)(x, 500, 0)
    # the runner stays usable after the error (flags are reset)
    x[0, 1, 7, 3] = 0.0
    eps = getattr(r, entry)(x, 500, 0)
    assert np.isfinite(eps).all()


def test_non_finite_x_T_in_sample_is_reported():
    # sample() -> the executor's require_finite on eps (proj/src/sampler.cpp:76-95)
    m = P.build_model(TINY, 97)
    cond = O.random_condition(8, 98)
    r = P.PatchRunner(m, cond, 16, 16, mode="displaced", n_devices=2, warmup_steps=1, dtype="bf16")
    x = O.random_normal(1, 2, 16, 16, 99)
    x[0, 0, 0, 0] = np.inf
    with pytest.raises(P.RuntimeFailure, match="non-finite value in tensor"):
        r.sample(x, P.make_plan(1000, 4), P.make_schedule(1000))


def test_full_size_1024_properties():
    # BASELINE configs[1] geometry (SDXL-shape, 128x128 latent = 1024^2 image), where the CPU
    # oracle is too slow for direct parity: size-independent properties instead.
    m = P.build_model(P.SDXL_SHAPE, 42)
    cond = P.random_condition(P.SDXL_SHAPE.cond_dim, 7)
    x_T = P.random_normal(1, 4, 128, 128, 1234)
    plan, abar = P.make_plan(1000, 3), P.make_schedule(1000)

    def run(mode, n, warmup=4):
        r = P.PatchRunner(m, cond, 128, 128, mode=mode, n_devices=n, warmup_steps=warmup,
                          dtype="bf16")
        a, _ = r.sample(x_T, plan, abar)
        b, _ = r.sample(x_T, plan, abar)          # graph replay
        assert np.array_equal(a, b)
        assert np.isfinite(a).all()
        return a

    ref = run("reference", 1)
    sync2 = run("sync-pp", 2)
    # every step synchronous (warm-up covers the run): displaced == sync-pp, bitwise
    assert np.array_equal(run("displaced", 2, warmup=3), sync2)
    # bands change only the GroupNorm statistics' combination order: bf16-level agreement
    assert rel(sync2, ref) <= TOL["bf16"]
    disp = run("displaced", 2, warmup=1)
    assert rel(disp, ref) <= 5e-2                 # one stale step at 1024^2


@pytest.mark.parametrize("mode,n,dtype", [("displaced", 2, "bf16"), ("sync-pp", 4, "fp32"),
                                          ("reference", 1, "bf16")])
def test_classifier_free_guidance_vs_oracle(mode, n, dtype):
    # cfg_scale (beyond the reference API): a second, unconditional
    # U-Net pass per step on its own band streams, eps = eps_u + s (eps_c - eps_u); per-step
    # latents against the oracle's two lockstep reference runners (run_sampling_cfg), graph
    # replay bitwise equal to the eager loop, both passes' MACs counted
    cfg = TOY
    m = P.build_model(cfg, 42)
    cond = O.random_condition(cfg.cond_dim, 7)
    unc = O.random_condition(cfg.cond_dim, 99)
    x = O.random_normal(1, cfg.in_channels, 32, 32, 1234)
    abar = O.make_schedule()
    plan = O.make_plan(1000, 4)
    r = P.PatchRunner(m, cond, 32, 32, mode=mode, n_devices=n, warmup_steps=1, dtype=dtype,
                      cfg_scale=3.0, uncond=unc)
    eager, traj = r.sample(x, plan, abar, trajectory=True)
    g, _ = r.sample(x, plan, abar)
    assert np.array_equal(g, eager)
    ref = O.run_sampling_cfg(ocfg(cfg), mode, n, 32, 32, 4, 1, cfg_scale=3.0, uncond=unc)
    for i in range(4):
        assert rel(traj[i], ref["trajectory"][i]) <= TOL[dtype], i
    assert rel(g, ref["x0"]) <= TOL[dtype]
    plain = O.run_sampling(ocfg(cfg), mode, n, 32, 32, 4, 1)["x0"]
    assert rel(plain, ref["x0"]) > 0.05                     # guidance really applied (7.8 %)
    assert r.total_macs() == 2 * ref["total_macs"]          # two sample() calls


def test_classifier_free_guidance_step_api_and_errors():
    # run_step with guidance returns the guided eps of the two passes (oracle: the two
    # reference runners' eps combined in fp64); uncond length and naive mode are checked
    cfg = TOY
    m = P.build_model(cfg, 42)
    cond = O.random_condition(cfg.cond_dim, 7)
    x = O.random_normal(1, cfg.in_channels, 32, 32, 1234)
    r = P.PatchRunner(m, cond, 32, 32, mode="sync-pp", n_devices=2, dtype="fp32", cfg_scale=2.5)
    eps = r.run_step(x, 700, 0)
    om = O.build_model(ocfg(cfg), 42)
    ec = O.PatchRunner(om, cond, 32, 32, "sync-pp", 2, 4, "corrected").run_step(x, 700, 0)
    eu = O.PatchRunner(om, np.zeros_like(cond), 32, 32, "sync-pp", 2, 4, "corrected").run_step(x, 700, 0)
    ref = (eu.astype(np.float64) + 2.5 * (ec.astype(np.float64) - eu)).astype(np.float32)
    assert rel(eps, ref) <= EPS_TOL["fp32"]
    with pytest.raises(P.InvalidArgument, match="uncond length"):
        P.PatchRunner(m, cond, 32, 32, mode="displaced", n_devices=2, cfg_scale=2.0,
                      uncond=np.zeros(cond.size + 1, np.float32))
    with pytest.raises(P.InvalidArgument, match="naive mode"):
        P.PatchRunner(m, cond, 32, 32, mode="naive", n_devices=2, cfg_scale=2.0)


def _oracle_run(cfg, cond, mode, n, hw, steps, warmup, seeds=(42, 1234)):
    """run_sampling (runtime.cpp:494-526) on the oracle with an explicit condition."""
    om = O.build_model(ocfg(cfg), seeds[0])
    r = O.PatchRunner(om, cond, hw, hw, mode, 1 if mode == "reference" else n, warmup, "corrected")
    counter = [0]

    def ex(x, t):
        e = r.run_step(x, t, counter[0])
        counter[0] += 1
        return e

    return O.sample(ex, O.make_plan(1000, steps), O.make_schedule(), 1, cfg.in_channels, hw, hw,
                    seeds[1])


@pytest.mark.parametrize("mode,n,dtype,tokens", [("displaced", 2, "bf16", 5), ("sync-pp", 4, "fp32", 77),
                                                 ("reference", 1, "bf16", 3)])
def test_multi_token_cross_attention_vs_oracle(mode, n, dtype, tokens):
    # layer_cross_attn (model.cpp:265-271) over T condition tokens (beyond the reference API,
    # which projects one): a 2-D condition [T][cond_dim]; the CrossAttn layer becomes a real
    # attention (S GEMM + softmax epilogue, rescale, PV GEMM) against the T projected rows
    cfg = TOY
    m = P.build_model(cfg, 42)
    cond = np.random.default_rng(tokens).standard_normal((tokens, cfg.cond_dim)).astype(np.float32)
    x = O.random_normal(1, cfg.in_channels, 32, 32, 1234)
    r = P.PatchRunner(m, cond, 32, 32, mode=mode, n_devices=n, warmup_steps=1, dtype=dtype)
    got, traj = r.sample(x, O.make_plan(1000, 4), O.make_schedule(), trajectory=True)
    g, _ = r.sample(x, O.make_plan(1000, 4), O.make_schedule())
    assert np.array_equal(g, got)
    ref, rtraj = _oracle_run(cfg, cond, mode, n, 32, 4, 1)
    for i in range(4):
        assert rel(traj[i], rtraj[i]) <= TOL[dtype], i
    assert rel(got, ref) <= TOL[dtype]
    single = _oracle_run(cfg, cond[0], mode, n, 32, 4, 1)[0]
    assert rel(single, ref) > 5e-3                    # the extra tokens matter


def test_multi_token_single_token_is_the_reference_path():
    # a [1][cond_dim] condition is exactly the reference's single-vector path
    cfg = TOY
    m = P.build_model(cfg, 42)
    cond = O.random_condition(cfg.cond_dim, 7)
    x = O.random_normal(1, cfg.in_channels, 32, 32, 1234)
    a = P.PatchRunner(m, cond, 32, 32, mode="displaced", n_devices=2, warmup_steps=1, dtype="bf16")
    b = P.PatchRunner(m, cond[None, :], 32, 32, mode="displaced", n_devices=2, warmup_steps=1,
                      dtype="bf16")
    plan, abar = O.make_plan(1000, 4), O.make_schedule()
    assert np.array_equal(a.sample(x, plan, abar)[0], b.sample(x, plan, abar)[0])
    with pytest.raises(P.InvalidArgument, match="condition: expected"):
        P.PatchRunner(m, np.zeros((3, cfg.cond_dim + 1), np.float32), 32, 32, mode="reference")


# two residual blocks per level and attention at levels 1 and 2 (4 self-attention layers at two
# geometries).  Deeper random-init stacks (attn_depth 2 + attn_up: residual-stream values of
# ~2e4, one-hot softmax rows) amplify bf16 / TF32 input rounding beyond the latent bar; their
# graph and weight pool are checked bit-exactly on the host (test_host_logic.py).
DEEP = dataclasses.replace(TOY, res_blocks=2, attn_levels=0b110)


@pytest.mark.parametrize("mode,n,dtype", [("displaced", 2, "bf16"), ("sync-pp", 4, "fp32"),
                                          ("reference", 1, "bf16")])
def test_deeper_graph_vs_oracle(mode, n, dtype):
    # a deeper U-Net (beyond the reference API): two residual blocks per level, attention at
    # levels 1 and 2; per-step latents against the oracle's runners over the same graph
    m = P.build_model(DEEP, 42)
    cond = O.random_condition(DEEP.cond_dim, 7)
    x = O.random_normal(1, DEEP.in_channels, 32, 32, 1234)
    r = P.PatchRunner(m, cond, 32, 32, mode=mode, n_devices=n, warmup_steps=1, dtype=dtype)
    got, traj = r.sample(x, O.make_plan(1000, 4), O.make_schedule(), trajectory=True)
    g, _ = r.sample(x, O.make_plan(1000, 4), O.make_schedule())
    assert np.array_equal(g, got)
    ref = O.run_sampling(ocfg(DEEP), mode, n, 32, 32, 4, 1)
    for i in range(4):
        assert rel(traj[i], ref["trajectory"][i]) <= TOL[dtype], i
    assert rel(got, ref["x0"]) <= TOL[dtype]
    assert r.total_macs() == 2 * ref["total_macs"]

"""Run artifacts (TNSR / PGM / psnr / weight pool, proj/src/io.cpp) and the CLI surface
(proj/src/cli.cpp): byte-compatibility with the reference build, error texts and exit codes."""
import ctypes as C
import os

import numpy as np
import pytest

from paper_2402_19481_b200 import artifacts as A
from paper_2402_19481_b200 import cli
from paper_2402_19481_b200 import patchsim as P


def _ref():
    from oracle import ref as R
    if not R.available():
        pytest.skip("oracle/_ref (reference build) not available")
    return R


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def test_tnsr_round_trip_bit_exact(tmp_path):
    x = np.random.default_rng(0).standard_normal((2, 3, 5, 7)).astype(np.float32)
    x[0, 0, 0, 0] = -0.0
    f = str(tmp_path / "x.tnsr")
    A.write_tnsr(x, f)
    y = A.read_tnsr(f)
    assert y.shape == x.shape and y.tobytes() == x.tobytes()
    blob = open(f, "rb").read()
    assert blob[:5] == b"TNSR\x01" and len(blob) == 4 + 1 + 4 + 16 + x.size * 4


@pytest.mark.parametrize("mutate,msg", [
    (lambda b: b"XNSR" + b[4:], "bad magic"),
    (lambda b: b[:4] + b"\x02" + b[5:], "unsupported version"),
    (lambda b: b[:5] + (3).to_bytes(4, "little") + b[9:], "expected 4 dims"),
    (lambda b: b[:-4], "payload shorter than dims"),
])
def test_tnsr_reader_errors(tmp_path, mutate, msg):
    f = str(tmp_path / "x.tnsr")
    A.write_tnsr(np.ones((1, 1, 2, 2), np.float32), f)
    blob = open(f, "rb").read()
    open(f, "wb").write(mutate(blob))
    with pytest.raises(P.RuntimeFailure, match=msg):
        A.read_tnsr(f)


def test_tnsr_rejects_non_finite(tmp_path):
    f = str(tmp_path / "x.tnsr")
    x = np.ones((1, 1, 2, 2), np.float32)
    x[0, 0, 1, 1] = np.inf
    A.write_tnsr(x, f)
    with pytest.raises(P.RuntimeFailure, match="non-finite"):
        A.read_tnsr(f)


def test_tnsr_pgm_psnr_match_reference(tmp_path):
    R = _ref()
    L = R.lib()
    x = np.random.default_rng(1).standard_normal((1, 4, 6, 9)).astype(np.float32)
    ours, theirs = str(tmp_path / "o.tnsr"), str(tmp_path / "t.tnsr")
    A.write_tnsr(x, ours)
    assert L.ref_write_tnsr(_p(x), 1, 4, 6, 9, theirs.encode()) == 0
    assert open(ours, "rb").read() == open(theirs, "rb").read()
    dims = np.zeros(4, np.int32)
    assert L.ref_read_tnsr_dims(ours.encode(), _p(dims)) == 0
    back = np.zeros(x.shape, np.float32)
    assert L.ref_read_tnsr(ours.encode(), _p(back)) == 0
    assert tuple(dims) == x.shape and back.tobytes() == x.tobytes()
    lo, hi = float(x.min()), float(x.max())
    A.write_pgm(x, str(tmp_path / "o.pgm"), lo, hi)
    assert L.ref_write_pgm(_p(x), 1, 4, 6, 9, C.c_double(lo), C.c_double(hi),
                           str(tmp_path / "t.pgm").encode()) == 0
    assert open(tmp_path / "o.pgm", "rb").read() == open(tmp_path / "t.pgm", "rb").read()
    A.write_pgm(np.zeros_like(x), str(tmp_path / "z.pgm"), 0.0, 0.0)   # zero range: mid-gray
    assert set(open(tmp_path / "z.pgm", "rb").read()[-x.size:]) == {128}
    y = x + 0.01 * np.random.default_rng(2).standard_normal(x.shape).astype(np.float32)
    L.ref_psnr.restype = C.c_double
    ref_db = L.ref_psnr(_p(x), _p(y), 1, 4, 6, 9, C.c_double(hi - lo))
    assert A.psnr(x, y, hi - lo) == pytest.approx(ref_db, rel=1e-12)
    assert A.psnr(x, x, 1.0) == float("inf")


def test_weight_pool_round_trip(tmp_path):
    cfg = P.ModelConfig()
    m = P.build_model(cfg, 5)
    f = str(tmp_path / "w.tnsr")
    A.dump_weights(m, f)
    m2 = A.load_weights(cfg, f)
    for a, b in zip(m.weights(), m2.weights()):
        assert a.tobytes() == b.tobytes()
    A.write_tnsr(np.ones((1, 1, 1, 7), np.float32), f)
    with pytest.raises(P.InvalidArgument, match="load_weights: file holds 7 values, model expects"):
        A.load_weights(cfg, f)


@pytest.mark.parametrize("argv,code", [
    (["--mode", "bogus"], 2),
    (["--emit", "video"], 2),
    (["--size", "30x30", "--devices", "4", "--mode", "sync-pp"], 2),   # RunConfig::validate
    (["--size", "abc"], 2),
    (["--no-such-flag"], 2),
    (["--compare-against", "/nonexistent/x0.tnsr"], 1),
])
def test_cli_error_exit_codes(tmp_path, argv, code):
    assert cli.run(argv + ["--out", str(tmp_path)]) == code


@pytest.mark.gpu
def test_cli_end_to_end(tmp_path):
    from oracle import patchsim_np as O
    ref = O.run_sampling(O.ModelConfig(), "displaced", 2, 32, 32, 4, 1)["x0"]
    rf = str(tmp_path / "ref.tnsr")
    A.write_tnsr(ref, rf)
    out = tmp_path / "out"
    code = cli.run(["--mode", "displaced", "--devices", "2", "--steps", "4", "--warmup", "1",
                    "--size", "32x32", "--out", str(out), "--compare-against", rf])
    assert code == 0
    x0 = A.read_tnsr(str(out / "x0.tnsr"))
    assert x0.shape == (1, 4, 32, 32)
    assert O.rel_l2(x0, ref) <= 2e-2
    assert A.read_tnsr(str(out / "trajectory.tnsr")).shape == (4, 4, 32, 32)
    metrics = dict(l.strip().split(",", 1) for l in open(out / "metrics.csv"))
    assert metrics["mode"] == "displaced" and metrics["devices"] == "2"
    assert float(metrics["psnr_db"]) > 30.0
    assert int(metrics["total_macs"]) > 0 and float(metrics["device_ms"]) > 0
    assert (out / "x0.pgm").exists() and (out / "trace.txt").exists()


def test_psnr_shape_mismatch_message():
    # require(a.same_shape(b), "psnr: shape mismatch " + a.shape_str() + ...) (tensor.cpp:337)
    a = np.zeros((1, 4, 6, 9), np.float32)
    b = np.zeros((1, 4, 6, 8), np.float32)
    with pytest.raises(P.InvalidArgument, match=r"^psnr: shape mismatch \(1,4,6,9\) vs \(1,4,6,8\)$"):
        A.psnr(a, b, 1.0)


def test_similarity_report_matches_reference_rule():
    # input_similarity_report (sampler.cpp:97-127): mean |x_t - x_{t-1}| over the pairs, range
    # over every state, ratio = mean / range
    traj = np.stack([np.full((1, 1, 2, 2), v, np.float32) for v in (0.0, 1.0, 3.0)])
    r = A.similarity_report(traj)
    assert r["per_step_mean_abs_diff"] == [1.0, 2.0]
    assert r["mean_abs_diff"] == 1.5 and (r["range_min"], r["range_max"]) == (0.0, 3.0)
    assert r["ratio"] == 0.5
    assert A.similarity_report(np.zeros((0, 1)))["ratio"] == 0.0
    assert A.similarity_report(np.zeros((3, 1, 2)))["ratio"] == 0.0


def test_cost_profile_parsing(tmp_path):
    # parse_cost_profile (io.cpp:110-131) + CostParams::validate (costmodel.cpp:13-19)
    f = tmp_path / "cost.txt"
    f.write_text("# comment\ncompute_rate = 2000\n\nlink_latency=1.5\n")
    p = A.parse_cost_profile(str(f))
    assert p == {"compute_rate": 2000.0, "link_bandwidth": 100.0, "link_latency": 1.5,
                 "comm_uses_compute_fraction": 0.15}
    for text, msg in (("bogus = 1", "unknown key 'bogus'"), ("compute_rate 3", "expected 'key = value'"),
                      ("link_bandwidth = 0", "rates must be positive"),
                      ("link_latency = -1", "negative latency"),
                      ("comm_uses_compute_fraction = 1", r"must be in \[0,1\)")):
        f.write_text(text + "\n")
        with pytest.raises(P.InvalidArgument, match=msg):
            A.parse_cost_profile(str(f))
    with pytest.raises(P.InvalidArgument, match="cannot open"):
        A.parse_cost_profile(str(tmp_path / "none.txt"))


def test_cli_config_and_matrix_files_are_validated(tmp_path):
    # --config 'key = value' mirroring the flags (cli.cpp:70), --matrix key=value rows
    # (cli.cpp:39-64): bad files are usage errors (exit 2) before any GPU work
    cfgf = tmp_path / "exp.cfg"
    cfgf.write_text("# base experiment\nmode = displaced\ndevices = 2\nsize = 32x32\nsteps = 4\n")
    assert cli.parse_config_file(str(cfgf)) == {"mode": "displaced", "devices": "2",
                                                "size": "32x32", "steps": "4"}
    cfgf.write_text("mode = displaced\nframes = 3\n")
    assert cli.run(["--config", str(cfgf), "--out", str(tmp_path)]) == 2
    base = {"mode": "reference", "devices": 1, "steps": 4, "warmup": 1, "size": "32x32",
            "model-seed": 42, "noise-seed": 1234, "cond-seed": 7, "gn-scheme": "corrected",
            "model": "toy", "dtype": "bf16"}
    mf = tmp_path / "runs.txt"
    mf.write_text("mode=displaced devices=2  # two bands\n\n# nothing\nmode=sync-pp devices=4 warmup=0\n")
    rows = cli.parse_matrix_file(base, str(mf))
    assert [(r["mode"], r["devices"]) for r in rows] == [("displaced", "2"), ("sync-pp", "4")]
    assert rows[1]["warmup"] == "0" and rows[0]["steps"] == 4
    for text, msg in (("mode=displaced frames=2", "unknown key 'frames'"),
                      ("displaced", "expected key=value"),
                      ("mode=sync-pp devices=3", "divisible")):
        mf.write_text(text + "\n")
        with pytest.raises(P.InvalidArgument, match=msg):
            cli.parse_matrix_file(base, str(mf))
        assert cli.run(["--matrix", str(mf), "--size", "32x32", "--out", str(tmp_path)]) == 2
    cost = tmp_path / "cost.txt"
    cost.write_text("link_bandwidth = -2\n")
    assert cli.run(["--cost-profile", str(cost), "--out", str(tmp_path)]) == 2


@pytest.mark.gpu
def test_cli_matrix_and_stress_sched(tmp_path):
    # run_matrix (io.cpp:288-328): one metrics row per experiment, psnr vs the matching
    # reference-mode run (inf for the reference row); --stress-sched must not change results
    mf = tmp_path / "runs.txt"
    mf.write_text("mode=reference\nmode=displaced devices=2 warmup=1\nmode=sync-pp devices=2\n")
    code = cli.run(["--matrix", str(mf), "--size", "32x32", "--steps", "4", "--out", str(tmp_path)])
    assert code == 0
    lines = open(tmp_path / "metrics.csv").read().splitlines()
    assert lines[0] == ("mode,N,steps,warmup,psnr_db_vs_reference,total_macs,per_device_macs,"
                        "comm_bytes,stall_us,makespan_us,similarity_ratio")
    rows = [l.split(",") for l in lines[1:]]
    assert [r[0] for r in rows] == ["reference", "displaced", "sync-pp"]
    assert rows[0][4] == "inf" and float(rows[1][4]) > 30.0 and float(rows[2][4]) > 40.0
    assert int(rows[0][7]) == 0 and int(rows[1][7]) > 0
    assert all(float(r[9]) > 0 and 0.0 < float(r[10]) < 1.0 for r in rows)
    outs = []
    for flag in ([], ["--stress-sched"]):
        d = tmp_path / ("s" if flag else "n")
        assert cli.run(["--mode", "displaced", "--devices", "2", "--steps", "4", "--warmup", "1",
                        "--size", "32x32", "--out", str(d), "--emit", "tensor"] + flag) == 0
        outs.append(A.read_tnsr(str(d / "x0.tnsr")))
    assert np.array_equal(outs[0], outs[1])

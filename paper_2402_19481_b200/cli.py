"""Command line of the B200 runner, mirroring the reference's ``patchsim`` CLI (proj/src/cli.cpp:
67-155) for one experiment: same flags, same artifacts (io.cpp:242-286), same exit codes
(0 ok, 2 invalid argument / usage, 1 runtime failure).

    python -m paper_2402_19481_b200.cli --mode displaced --devices 2 --steps 50 --warmup 4 \\
        --size 48x48 --out out [--compare-against ref_x0.tnsr] [--emit tensor metrics ...]
    python -m paper_2402_19481_b200.cli --config exp.cfg --matrix runs.txt --out out

--config (cli.cpp:70): a plain 'key = value' file mirroring the flags (command-line flags
win).  --matrix (cli.cpp:106-107, 131-139; io.cpp:288-328): one experiment per line of
key=value overrides (mode devices steps warmup size model-seed noise-seed cond-seed
gn-scheme), every non-reference row compared against the matching reference-mode run;
writes out/metrics.csv with the reference's columns.  --stress-sched (cli.cpp:104;
collectives.cpp:45-56): seeded sleep kernels around every exchange; results unchanged.
--cost-profile (cli.cpp:96; io.cpp:110-131): parsed and validated like the reference; the
simulated timeline it parameterises is out of scope, so it is only echoed
into metrics.csv.

Differences, by design: the sampling runs on the B200 runner (`patchsim.PatchRunner.sample`,
every band on this process's GPU(s)); `trace.txt` holds the RawTrace events (the reference
writes the cost model's simulated timeline, which is out of scope here);
`metrics.csv` reports the measured device time (`device_ms`) where the reference reports its
simulated `makespan_us` / `stall_us`, and the bytes this runtime actually exchanged
(`comm_bytes_*`).  `--model sdxl` selects the SDXL-shape config, `--dtype`
the arithmetic."""
from __future__ import annotations

import argparse
import math
import os
import sys

import numpy as np

from . import artifacts as A
from . import patchsim as P

ARTIFACTS = ("image", "tensor", "trace", "metrics")


def _fmt(v: float) -> str:
    """fmt (io.cpp:31-36): %.6g."""
    return "%.6g" % v


def parse_size(s: str):
    """parse_size (cli.cpp): 'HxW'."""
    try:
        h, w = s.lower().split("x")
        return int(h), int(w)
    except ValueError:
        raise P.InvalidArgument(f"--size: expected HxW, got '{s}'") from None


CONFIG_KEYS = ("mode", "devices", "steps", "warmup", "size", "model-seed", "noise-seed",
               "cond-seed", "out", "compare-against", "cost-profile", "emit", "gn-scheme",
               "stress-sched", "matrix", "model", "dtype", "weights", "cfg-scale", "cond-tokens")
MATRIX_KEYS = ("mode", "devices", "steps", "warmup", "size", "model-seed", "noise-seed",
               "cond-seed", "gn-scheme")


def parse_config_file(path: str) -> dict:
    """--config: 'key = value' lines (CLI11 config file; '#' / ';' comments, [sections]
    ignored), keys = the long flag names.  Unknown keys are InvalidArgument (exit 2)."""
    try:
        f = open(path)
    except OSError:
        raise P.InvalidArgument(f"--config: cannot open {path}") from None
    out = {}
    with f:
        for line in f:
            t = line.strip()
            if not t or t[0] in "#;" or (t.startswith("[") and t.endswith("]")):
                continue
            if "=" not in t:
                raise P.InvalidArgument(f"--config: expected 'key = value', got '{t}'")
            k, v = (x.strip() for x in t.split("=", 1))
            k = k.lstrip("-")
            if k not in CONFIG_KEYS:
                raise P.InvalidArgument(f"--config: unknown key '{k}'")
            v = v.strip('"')
            if k == "emit":
                out[k] = [e for e in v.replace(",", " ").split() if e]
            elif k == "stress-sched":
                out[k] = v.lower() in ("1", "true", "yes", "on")
            else:
                out[k] = v
    return out


def parse_matrix_file(base: dict, path: str):
    """parse_matrix_file (cli.cpp:39-64): each non-empty line = key=value overrides of the
    base experiment; '#' starts a comment; every row is validated."""
    try:
        f = open(path)
    except OSError:
        raise P.InvalidArgument(f"matrix: cannot open {path}") from None
    rows = []
    with f:
        for line in f:
            cfg = dict(base)
            any_ = False
            for tok in line.split():
                if tok.startswith("#"):
                    break
                if "=" not in tok:
                    raise P.InvalidArgument(f"matrix: expected key=value, got '{tok}'")
                k, v = tok.split("=", 1)
                if k not in MATRIX_KEYS:
                    raise P.InvalidArgument(f"matrix: unknown key '{k}'")
                cfg[k] = v
                any_ = True
            if any_:
                _run_config(cfg).validate()
                rows.append(cfg)
    return rows


def _run_config(e: dict):
    if e["mode"] not in P.N.MODES:
        raise P.InvalidArgument(f"unknown run mode '{e['mode']}'")
    if e["gn-scheme"] not in P.N.GN_SCHEMES:
        raise P.InvalidArgument(f"unknown GroupNorm scheme '{e['gn-scheme']}'")
    h, w = parse_size(e["size"])
    mcfg = P.SDXL_SHAPE if e["model"] == "sdxl" else P.ModelConfig()
    try:
        return P.RunConfig(mode=e["mode"], n_devices=int(e["devices"]), h=h, w=w,
                           num_steps=int(e["steps"]), warmup=int(e["warmup"]),
                           gn_scheme=e["gn-scheme"], dtype=e["dtype"],
                           model_seed=int(e["model-seed"]), noise_seed=int(e["noise-seed"]),
                           cond_seed=int(e["cond-seed"]), model=mcfg)
    except ValueError as err:
        raise P.InvalidArgument(f"bad value: {err}") from None


def _execute(rc, stress=False, trajectory=False, no_comm=False, weights=""):
    """execute_experiment (io.cpp) on the B200 runner: x0, trajectory, runner stats."""
    mcfg = rc.model
    model = A.load_weights(mcfg, weights) if weights else P.build_model(mcfg, rc.model_seed)
    cond = P.random_condition(mcfg.cond_dim, rc.cond_seed)
    x_T = P.random_normal(1, mcfg.in_channels, rc.h, rc.w, rc.noise_seed)
    abar = P.make_schedule(rc.schedule_steps, rc.beta_start, rc.beta_end)
    plan = P.make_plan(rc.schedule_steps, rc.num_steps)
    n = 1 if rc.mode == "reference" else rc.n_devices
    runner = P.PatchRunner(model, cond, rc.h, rc.w, mode=rc.mode, n_devices=n,
                           warmup_steps=rc.warmup, gn_scheme=rc.gn_scheme, dtype=rc.dtype,
                           stress=stress, no_comm=no_comm)
    x0, traj = runner.sample(x_T, plan, abar, trajectory=trajectory)
    vol = runner.volumes()
    out = {"x0": x0, "trajectory": traj, "device_ms": runner.last_device_ms(),
           "total_macs": runner.total_macs(),
           "per_device_macs": max(runner.step_device_macs(0)) * rc.num_steps if rc.num_steps else 0,
           "volumes": vol,
           "comm_bytes": vol["allgather_recv"] + vol["halo_recv"] + vol["statreduce_recv"],
           "runner": runner}
    return out


def run_matrix(rows, stress=False) -> str:
    """run_matrix (io.cpp:288-328) with measured columns: makespan_us = the run's device
    time; stall_us = its exposed communication, T - T(no exchange) on the same bands (the
    paper's "No Comm." ablation, 0 without an exchange); the reference-mode x0 is cached per
    (size, steps, seeds, model)."""
    lines = ["mode,N,steps,warmup,psnr_db_vs_reference,total_macs,per_device_macs,comm_bytes,"
             "stall_us,makespan_us,similarity_ratio"]
    refs = {}
    for e in rows:
        rc = _run_config(e)
        out = _execute(rc, stress=stress, trajectory=True)
        sim = A.similarity_report(out["trajectory"])["ratio"]
        if rc.mode == "reference":
            psnr = math.inf
        else:
            key = (rc.h, rc.w, rc.num_steps, rc.model_seed, rc.noise_seed, rc.cond_seed,
                   e["model"], e["dtype"])
            if key not in refs:
                rr = _run_config({**e, "mode": "reference", "devices": "1"})
                refs[key] = _execute(rr)["x0"]
            ref = refs[key]
            psnr = A.psnr(out["x0"], ref, float(np.max(ref)) - float(np.min(ref)))
        stall = 0.0
        if rc.mode in ("sync-pp", "displaced") and rc.n_devices > 1:
            t_nc = _execute(rc, no_comm=True)["device_ms"]
            stall = max(0.0, out["device_ms"] - t_nc) * 1e3
        n = 1 if rc.mode == "reference" else rc.n_devices
        lines.append(",".join([rc.mode, str(n), str(rc.num_steps), str(rc.warmup), _fmt(psnr),
                               str(out["total_macs"]), str(out["per_device_macs"]),
                               str(out["comm_bytes"]), _fmt(stall),
                               _fmt(out["device_ms"] * 1e3), _fmt(sim)]))
    return "\n".join(lines) + "\n"


def build_parser():
    ap = argparse.ArgumentParser(prog="patchsim-b200",
                                 description="Patch-parallel diffusion inference on B200")
    ap.add_argument("--mode", default="reference", help="reference|naive|sync-pp|displaced")
    ap.add_argument("--devices", type=int, default=1, help="patch (band) count")
    ap.add_argument("--steps", type=int, default=50, help="denoising steps")
    ap.add_argument("--warmup", type=int, default=4, help="synchronous warm-up steps (displaced)")
    ap.add_argument("--size", default="48x48", help="latent size HxW")
    ap.add_argument("--model-seed", type=int, default=42)
    ap.add_argument("--noise-seed", type=int, default=1234)
    ap.add_argument("--cond-seed", type=int, default=7)
    ap.add_argument("--out", default="out", help="output directory")
    ap.add_argument("--compare-against", default="", help="x0 TNSR for PSNR")
    ap.add_argument("--emit", nargs="*", default=None, help="image tensor trace metrics")
    ap.add_argument("--gn-scheme", default="corrected", help="corrected|stale|separate")
    ap.add_argument("--model", default="toy", choices=["toy", "sdxl"])
    ap.add_argument("--dtype", default="bf16", choices=["bf16", "fp32"])
    ap.add_argument("--weights", default="", help="TNSR weight pool (dump_weights order)")
    ap.add_argument("--config", default="", help="'key = value' file mirroring the flags")
    ap.add_argument("--cost-profile", default="", help="cost model 'key = value' file")
    ap.add_argument("--stress-sched", action="store_true",
                    help="inject scheduling noise around the exchanges (determinism check)")
    ap.add_argument("--matrix", default="", help="experiment list; each line key=value overrides")
    ap.add_argument("--cfg-scale", type=float, default=0.0,
                    help="classifier-free guidance scale (0 = off; unconditional = zeros)")
    ap.add_argument("--cond-tokens", type=int, default=1,
                    help="condition tokens (random_condition over tokens x cond_dim)")
    return ap


def run(argv) -> int:
    ap = build_parser()
    try:
        pre, _ = ap.parse_known_args(argv)
    except SystemExit as e:
        return 0 if e.code == 0 else 2
    try:
        if pre.config:
            # config values become defaults: flags given on the command line win (CLI11)
            ap.set_defaults(**{k.replace("-", "_"): v for k, v in parse_config_file(pre.config).items()})
    except P.InvalidArgument as e:
        print(f"error: {e}", file=sys.stderr)
        return 2
    try:
        args = ap.parse_args(argv)
        args.devices, args.steps, args.warmup = int(args.devices), int(args.steps), int(args.warmup)
        args.model_seed, args.noise_seed = int(args.model_seed), int(args.noise_seed)
        args.cond_seed = int(args.cond_seed)
        args.cfg_scale, args.cond_tokens = float(args.cfg_scale), int(args.cond_tokens)
    except SystemExit as e:
        return 0 if e.code == 0 else 2
    except ValueError as e:
        print(f"error: {e}", file=sys.stderr)
        return 2
    try:
        if args.mode not in P.N.MODES:
            raise P.InvalidArgument(f"unknown run mode '{args.mode}'")
        if args.gn_scheme not in P.N.GN_SCHEMES:
            raise P.InvalidArgument(f"unknown GroupNorm scheme '{args.gn_scheme}'")
        emit = ARTIFACTS if args.emit is None else tuple(args.emit)
        for e in emit:
            if e not in ARTIFACTS:
                raise P.InvalidArgument(f"--emit: unknown artifact '{e}'")
        cost = A.parse_cost_profile(args.cost_profile) if args.cost_profile else None
        if args.matrix:
            base = {"mode": args.mode, "devices": args.devices, "steps": args.steps,
                    "warmup": args.warmup, "size": args.size, "model-seed": args.model_seed,
                    "noise-seed": args.noise_seed, "cond-seed": args.cond_seed,
                    "gn-scheme": args.gn_scheme, "model": args.model, "dtype": args.dtype}
            rows = parse_matrix_file(base, args.matrix)
            csv = run_matrix(rows, stress=args.stress_sched)
            os.makedirs(args.out, exist_ok=True)
            with open(os.path.join(args.out, "metrics.csv"), "w") as f:
                f.write(csv)
            return 0
        h, w = parse_size(args.size)
        mcfg = P.SDXL_SHAPE if args.model == "sdxl" else P.ModelConfig()
        rc = P.RunConfig(mode=args.mode, n_devices=args.devices, h=h, w=w, num_steps=args.steps,
                         warmup=args.warmup, gn_scheme=args.gn_scheme, dtype=args.dtype,
                         model_seed=args.model_seed, noise_seed=args.noise_seed,
                         cond_seed=args.cond_seed, model=mcfg)
        rc.validate()   # RunConfig::validate (runtime.cpp:480-492), before any GPU work
        ref = A.read_tnsr(args.compare_against) if args.compare_against else None

        model = (A.load_weights(mcfg, args.weights) if args.weights
                 else P.build_model(mcfg, args.model_seed))
        if args.cond_tokens < 1:
            raise P.InvalidArgument("--cond-tokens must be >= 1")
        cond = P.random_condition(mcfg.cond_dim * args.cond_tokens, args.cond_seed)
        if args.cond_tokens > 1:
            cond = cond.reshape(args.cond_tokens, mcfg.cond_dim)
        x_T = P.random_normal(1, mcfg.in_channels, h, w, args.noise_seed)
        abar = P.make_schedule(rc.schedule_steps, rc.beta_start, rc.beta_end)
        plan = P.make_plan(rc.schedule_steps, args.steps)
        runner = P.PatchRunner(model, cond, h, w, mode=args.mode, n_devices=args.devices,
                               warmup_steps=args.warmup, gn_scheme=args.gn_scheme,
                               dtype=args.dtype, stress=args.stress_sched, cfg_scale=args.cfg_scale)
        x0, traj = runner.sample(x_T, plan, abar, trajectory="tensor" in emit)
        device_ms = runner.last_device_ms()

        os.makedirs(args.out, exist_ok=True)
        d = args.out
        lo, hi = float(np.min(x0)), float(np.max(x0))
        if "tensor" in emit:
            A.write_tnsr(x0, os.path.join(d, "x0.tnsr"))
            if traj is not None:
                t = np.asarray(traj, dtype=np.float32)
                A.write_tnsr(t.reshape(-1, *t.shape[-3:]), os.path.join(d, "trajectory.tnsr"))
        if "image" in emit:
            A.write_pgm(x0, os.path.join(d, "x0.pgm"), lo, hi)
        if "trace" in emit:
            with open(os.path.join(d, "trace.txt"), "w") as f:
                f.write("device,step,layer,kind,prim,macs,bytes_recv,bytes_sent,tag\n")
                for dev in range(runner.n_devices):
                    for ev in runner.trace(dev):
                        f.write(",".join(str(v) for v in ev) + "\n")
        if "metrics" in emit:
            vol = runner.volumes()
            per_dev = max(runner.step_device_macs(0)) * args.steps if args.steps else 0
            rows = [("mode", args.mode), ("devices", args.devices), ("steps", args.steps),
                    ("warmup", args.warmup), ("gn_scheme", args.gn_scheme)]
            if ref is not None:
                peak = float(np.max(ref)) - float(np.min(ref))
                rows += [("psnr_db", _fmt(A.psnr(x0, ref, peak))), ("psnr_peak", _fmt(peak))]
            recv = vol["allgather_recv"] + vol["halo_recv"] + vol["statreduce_recv"]
            rows += [("output_min", _fmt(lo)), ("output_max", _fmt(hi)),
                     ("total_macs", runner.total_macs()), ("per_device_macs", per_dev),
                     ("comm_bytes_allgather", vol["allgather_recv"]),
                     ("comm_bytes_halo", vol["halo_recv"]),
                     ("comm_bytes_statreduce", vol["statreduce_recv"]),
                     ("comm_bytes_total", recv), ("device_ms", _fmt(device_ms))]
            if traj is not None:
                rows.append(("similarity_ratio", _fmt(A.similarity_report(traj)["ratio"])))
            if cost is not None:
                rows += [("cost_" + k, _fmt(v)) for k, v in cost.items()]
            if args.stress_sched:
                rows.append(("stress_sched", 1))
            with open(os.path.join(d, "metrics.csv"), "w") as f:
                f.write("metric,value\n")
                for k, v in rows:
                    f.write(f"{k},{v}\n")
        return 0
    except P.InvalidArgument as e:
        print(f"error: {e}", file=sys.stderr)
        return 2
    except Exception as e:  # noqa: BLE001  (reference: std::exception -> exit 1)
        print(f"error: {e}", file=sys.stderr)
        return 1


def main():
    sys.exit(run(sys.argv[1:]))


if __name__ == "__main__":
    main()

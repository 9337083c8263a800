"""Command line of the B200 runner, mirroring the reference's ``patchsim`` CLI (proj/src/cli.cpp:
67-155) for one experiment: same flags, same artifacts (io.cpp:242-286), same exit codes
(0 ok, 2 invalid argument / usage, 1 runtime failure).

    python -m paper_2402_19481_b200.cli --mode displaced --devices 2 --steps 50 --warmup 4 \\
        --size 48x48 --out out [--compare-against ref_x0.tnsr] [--emit tensor metrics ...]

Differences, by design: the sampling runs on the B200 runner (`patchsim.PatchRunner.sample`,
every band on this process's GPU(s)); `trace.txt` holds the RawTrace events (the reference
writes the cost model's simulated timeline, which is out of scope here);
`metrics.csv` reports the measured device time (`device_ms`) where the reference reports its
simulated `makespan_us` / `stall_us`, and the bytes this runtime actually exchanged
(`comm_bytes_*`).  `--model sdxl` selects the SDXL-shape config, `--dtype`
the arithmetic."""
from __future__ import annotations

import argparse
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
    return ap


def run(argv) -> int:
    ap = build_parser()
    try:
        args = ap.parse_args(argv)
    except SystemExit as e:
        return 0 if e.code == 0 else 2
    try:
        if args.mode not in P.N.MODES:
            raise P.InvalidArgument(f"unknown run mode '{args.mode}'")
        if args.gn_scheme not in P.N.GN_SCHEMES:
            raise P.InvalidArgument(f"unknown GroupNorm scheme '{args.gn_scheme}'")
        emit = ARTIFACTS if args.emit is None else tuple(args.emit)
        for e in emit:
            if e not in ARTIFACTS:
                raise P.InvalidArgument(f"--emit: unknown artifact '{e}'")
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
        cond = P.random_condition(mcfg.cond_dim, args.cond_seed)
        x_T = P.random_normal(1, mcfg.in_channels, h, w, args.noise_seed)
        abar = P.make_schedule(rc.schedule_steps, rc.beta_start, rc.beta_end)
        plan = P.make_plan(rc.schedule_steps, args.steps)
        runner = P.PatchRunner(model, cond, h, w, mode=args.mode, n_devices=args.devices,
                               warmup_steps=args.warmup, gn_scheme=args.gn_scheme,
                               dtype=args.dtype)
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

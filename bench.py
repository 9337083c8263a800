#!/usr/bin/env python3
"""Headline benchmark: SDXL-shape 50-step sampling latency on B200 (BASELINE.json metric).

One "step" of this benchmark = one full 50-step DDIM-eta0 (== Euler in sigma space)
generation of an SDXL-shape latent through the displaced-patch-parallel runtime
(configs[1]: 1024x1024 image, 128x128 latent; N = 1, 2, 4, 8 GPUs, one rank per GPU).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
  (N > 1: python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N)

value      device latency of one generation (CUDA events on the runtime's own compute
           streams, x_T already resident; max over ranks), seconds, lower is better
e2e        the same generation through the public C ABI (pp_runner_sample) from a host
           x_T to a host x0, wall clock around the synchronous call (max over ranks)
roofline   dominant kernel = the tcgen05 implicit-GEMM conv; algorithmic FLOPs
           (2 * macs_of_layer, proj/src/costmodel.cpp:33-62) / CUDA-event kernel time
cpu_baseline  the reference's own CPU path (oracle/_ref = /root/reference/proj/src built
           unmodified) on this box's host cores: a bounded sample (one sync-pp step over
           4 thread bands at a 48x48 latent), extrapolated to the workload by MAC count
           (optimistic for the CPU: its per-MAC cost grows with the latent size)
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

os.environ.setdefault("OMP_NUM_THREADS", str(os.cpu_count() or 1))
ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "SDXL-shape 50-step latency (s) & speedup at 1/2/4/8 B200, 1024²–3840²"
SDXL = (4, 320, 3, 32, 2048, -1)
SEEDS = (42, 1234, 7)   # model, noise, condition (RunConfig defaults, runtime.hpp:121-123)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--latent", type=int, default=128, help="latent side (image = 8x)")
    ap.add_argument("--latent-w", type=int, default=0,
                    help="latent width when not square (e.g. 160x240 = 1280x1920 image)")
    ap.add_argument("--num-steps", type=int, default=50)
    ap.add_argument("--mode", default="displaced")
    ap.add_argument("--warmup-steps", type=int, default=4, help="displaced: sync warm-up steps")
    ap.add_argument("--dtype", default="bf16", choices=["bf16", "fp32"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--transport", default="nccl", choices=["nccl", "ipc"],
                    help="N>1 (torchrun): NCCL, or CUDA IPC peer buffers + copy engines")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def workload(args, n):
    return {
        "workload": f"SDXL-shape UNet (4->320/640/1280 ch, GN32, d=1280 self-attn, 77.4M params, "
                    f"random init seed 42), {8 * args.latent}x{8 * (args.latent_w or args.latent)} image "
                    f"({args.latent}x{args.latent_w or args.latent} latent), {args.num_steps}-step DDIM-eta0 "
                    f"(Euler) sampling, displaced patch parallelism over {n} row band(s), "
                    f"{args.warmup_steps} synchronous warm-up steps",
        "latent": [args.latent, args.latent_w or args.latent],
        "sampling_steps": args.num_steps,
        "mode": args.mode if n > 1 else "displaced (N=1: identical to reference mode)",
        "patches": n,
        "parallelism": f"pp{n}",
        **({"transport": args.transport} if n > 1 and os.environ.get("WORLD_SIZE", "1") != "1" else {}),
        "l2": "flushed between timed generations (256 MiB device write)",
        "timed_unit": "one full generation (x_T -> x0)",
    }


# ------------------------------------------------------------------------ reference CPU path
def cpu_threads():
    """Bands for the threaded reference sample: a power of two <= host cores, <= 4 (the
    reference's sync-pp step stops scaling beyond ~4 threads: per-layer hub barriers)."""
    n = 1
    while n * 2 <= min(os.cpu_count() or 1, 4):
        n *= 2
    return n


def cpu_reference_sample(latent_full, num_steps):
    """Time one step of the reference's own CPU path (oracle/_ref, unmodified
    proj/src sources) on a 48x48 SDXL-shape latent and extrapolate by MAC count to
    `num_steps` steps at latent_full^2.  The reference's only multi-threaded execution is
    its PatchRunner (one std::thread per simulated device, runtime.cpp:337-380; tensor ops
    are single-threaded), so the step is a synchronous patch-parallel step (sync-pp: same
    result as the reference forward, test_runtime.cpp:231-248) over cpu_threads() bands --
    every host core busy."""
    from oracle import ref as R
    if not os.path.exists(R.LIB_PATH) and not os.path.isdir(R.REF_SRC):
        return None
    model = R.Model(SDXL, SEEDS[0])
    cond = R.random_condition(2048, SEEDS[2])
    side = 48
    n = cpu_threads()
    x = R.random_normal(1, 4, side, side, SEEDS[1])
    runner = R.PatchRunner(model, cond, side, side, mode="sync-pp" if n > 1 else "reference",
                           n_devices=n)
    t0 = time.perf_counter()
    runner.step("run_step", x, 980, 0)
    dt = time.perf_counter() - t0
    scale = model.total_macs(latent_full, latent_full) / model.total_macs(side, side)
    return {"seconds_sample": dt, "value": dt * scale * num_steps, "macs_ratio": scale,
            "sample": f"1 denoising step of the reference CPU path (PatchRunner::run_step, "
                      f"proj/src/runtime.cpp:454-476, {'sync-pp over ' + str(n) + ' thread bands' if n > 1 else 'reference mode'}) "
                      f"on the SDXL-shape model at a {side}x{side} latent, extrapolated "
                      f"x{scale:.2f} by model_total_macs to {latent_full}x{latent_full} and "
                      f"x{num_steps} steps",
            "kind": "reference", "cores": n}


def cpu_port_sample(latent_full, num_steps):
    """Fallback when oracle/_ref is absent: the numpy restatement (oracle/patchsim_np.py)."""
    from oracle import patchsim_np as O
    m = O.build_model(O.SDXL_SHAPE, SEEDS[0])
    cond = O.random_condition(2048, SEEDS[2])
    side = 32
    x = O.random_normal(1, 4, side, side, SEEDS[1])
    t0 = time.perf_counter()
    O.forward_full(m, x, 980, cond)
    dt = time.perf_counter() - t0
    scale = O.model_total_macs(m, latent_full, latent_full) / O.model_total_macs(m, side, side)
    return {"seconds_sample": dt, "value": dt * scale * num_steps, "macs_ratio": scale,
            "sample": f"1 reference-mode step of the numpy port at {side}x{side}, extrapolated "
                      f"x{scale:.2f} by MACs and x{num_steps} steps",
            "kind": "port", "cores": os.cpu_count() or 1}


def run_reference_arm(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    try:
        probe = cpu_reference_sample
        from oracle import ref as R
        if not os.path.exists(R.LIB_PATH) and not os.path.isdir(R.REF_SRC):
            probe = cpu_port_sample
    except Exception:
        probe = cpu_port_sample
    for _ in range(args.warmup):
        probe(args.latent, args.num_steps)
    samples = [probe(args.latent, args.num_steps) for _ in range(args.steps)]
    v = statistics.mean(s["value"] for s in samples)
    s0 = samples[0]
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": v * 1e3,
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded splitmix64 weights / Box-Muller latent, as the reference)",
        "config": workload(args, 1),
        "cpu_baseline": {"value": v, "unit": "s", "cores": s0["cores"], "kind": s0["kind"],
                         "sample": s0["sample"] + "; each timed step is one such sample"},
        "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------ clocks
class ClockSampler:
    def __init__(self, gpu):
        self.gpu = gpu
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.thread:
            self.thread.join(timeout=5)
        sm = [float(r[1]) for r in self.rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            if len(r) < 9:
                continue
            for k, nm in enumerate(names):
                if r[5 + k].lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------------ our arm
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference_arm(args)
    world, rank, local = dist_env()
    import torch
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2402_19481_b200 import patchsim as P

    n = world if world > 1 else args.gpus
    if world == 1 and n > 1 and torch.cuda.device_count() < n:
        n = args.gpus   # in-process bands share the visible devices
    nccl_id = None
    if world > 1 and args.transport == "nccl":
        obj = [P.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]

    model = P.build_model(P.ModelConfig(*SDXL), SEEDS[0])
    cond = P.random_condition(2048, SEEDS[2])
    H, W = args.latent, (args.latent_w or args.latent)
    runner = P.PatchRunner(model, cond, H, W, mode=args.mode if n > 1 else "displaced",
                           n_devices=n, warmup_steps=args.warmup_steps, dtype=args.dtype,
                           world=world, rank=rank, nccl_id=nccl_id, device=local,
                           transport=args.transport)
    if world > 1 and args.transport == "ipc":
        runner.connect_ipc()
    abar = P.make_schedule(1000)
    plan = P.make_plan(1000, args.num_steps)
    x_T = P.random_normal(1, 4, H, W, SEEDS[1])
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()

    for _ in range(args.warmup):
        runner.sample(x_T, plan, abar)
    barrier()
    clocks = ClockSampler(local)
    clocks.start()
    dev_ms, wall_s, launches = [], [], 0
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        x0, _ = runner.sample(x_T, plan, abar)
        wall_s.append(time.perf_counter() - t0)
        dev_ms.append(runner.last_device_ms())
        launches += runner.launches()
    barrier()
    clk = clocks.stop()

    dev = statistics.mean(dev_ms) / 1e3
    e2e = statistics.mean(wall_s)
    if dist is not None:
        t = torch.tensor([dev, e2e], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dev, e2e = float(t[0]), float(t[1])

    # instrumented pass (outside the timed region): per-kernel CUDA events
    runner.set_profile(True)
    runner.sample(x_T, plan, abar)
    prof = runner.profile()
    runner.set_profile(False)
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except Exception:
        pass
    peak = float(peaks.get("bf16_tflops_sustained", 1380.4))
    peak_src = "measured (MEASURED_PEAKS.json bf16_tflops_sustained)" if peaks else "fallback 1400"
    achieved = prof["conv_flops"] / (prof["conv_ms"] / 1e3) / 1e12 if prof["conv_ms"] else None
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            traffic = json.load(f).get("conv_dram_bytes_per_launch")
    except Exception:
        pass
    n_conv = prof.get("launches", 0)
    roofline = {
        "bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
        "frac": (achieved / peak) if achieved else None, "traffic": traffic,
        "kernel": "gemm_kernel<bf16> (tcgen05 implicit-GEMM 3x3 conv, all conv layers)",
        "peak_source": peak_src,
        "conv_ms_per_generation": prof["conv_ms"],
        "gemm_ms_per_generation": prof["gemm_ms"], "gn_ms_per_generation": prof["gn_ms"],
        "other_ms_per_generation": prof["other_ms"],
        "conv_share_of_step": prof["conv_ms"] / (dev * 1e3) if dev else None,
    }

    cpu = None
    if rank == 0 and world == 1 and n == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_reference_sample(args.latent, args.num_steps) or cpu_port_sample(
                args.latent, args.num_steps)
        except Exception as e:  # report, never fake
            cpu = {"value": None, "error": str(e)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": dev, "unit": "s", "n_gpus": n, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dev * 1e3, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": args.dtype,
            "data": "synthetic (seeded random-init SDXL-shape weights, Box-Muller x_T)",
            "config": workload(args, n),
            "e2e": {"value": e2e, "unit": "s", "h2d_bytes_per_step": int(x_T.nbytes),
                    "d2h_bytes_per_step": int(x_T.nbytes),
                    "path": "pp_runner_sample C ABI, host x_T in / host x0 out"},
            "gpu_launches": launches,
            "roofline": roofline,
            "clocks": clk,
        }
        if cpu is not None:
            line["cpu_baseline"] = {"value": cpu.get("value"), "unit": "s",
                                    "cores": cpu.get("cores"), "kind": cpu.get("kind"),
                                    "sample": cpu.get("sample"),
                                    "seconds_per_sample": cpu.get("seconds_sample")}
        print(json.dumps(line), flush=True)
    runner.close()
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())

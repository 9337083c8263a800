"""Worker of tests/test_ipc_gpu.py: one rank of a world-2 / world-4 run with the copy-engine
(CUDA IPC) transport, or the NCCL transport when argv[2] == "nccl", all ranks on cuda:0 (the
pool has one GPU per box; CUDA IPC maps a buffer of another process on the same device exactly
as on a peer).  Rank 0 repeats the run in-process
(world 1, two bands: the in-process transport, itself parity-tested against the oracle) and
writes the comparison to argv[1]."""
import json
import os
import sys

TRANSPORT = sys.argv[2] if len(sys.argv) > 2 else "ipc"
if TRANSPORT == "nccl":
    # NCCL refuses two ranks of one host on one device ("Duplicate GPU"); a distinct
    # NCCL_HOSTID per rank makes them look like separate hosts, so NCCL connects them over its
    # socket transport (loopback): slow, but the NCCL transport's real code path runs
    os.environ["NCCL_HOSTID"] = "pp-test-host-" + os.environ.get("RANK", "0")
    os.environ.setdefault("NCCL_SOCKET_IFNAME", "lo")
    os.environ.setdefault("NCCL_IB_DISABLE", "1")

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2402_19481_b200 import patchsim as P  # noqa: E402


def main():
    import faulthandler
    faulthandler.dump_traceback_later(240, exit=True)   # a hang reports where it is, then exits
    out_path = sys.argv[1]
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    cfg = P.ModelConfig()
    h = w = 32
    steps = 6
    model = P.build_model(cfg, 42)
    cond = P.random_condition(cfg.cond_dim, 7)
    x_T = P.random_normal(1, cfg.in_channels, h, w, 1234)
    abar = P.make_schedule(1000)
    plan = P.make_plan(1000, steps)
    res = {}
    for mode, warmup in (("displaced", 1), ("sync-pp", 0), ("displaced", 0)):
        for dtype in ("bf16", "fp32"):
            kw = {}
            if TRANSPORT == "nccl":
                ids = [P.nccl_unique_id() if rank == 0 else None]
                dist.broadcast_object_list(ids, 0)
                kw["nccl_id"] = ids[0]
            r = P.PatchRunner(model, cond, h, w, mode=mode, n_devices=world, warmup_steps=warmup,
                              dtype=dtype, world=world, rank=rank, device=0, transport=TRANSPORT,
                              **kw)
            if TRANSPORT == "ipc":
                r.connect_ipc()
            x0, _ = r.sample(x_T, plan, abar)
            x0b, traj = r.sample(x_T, plan, abar, trajectory=True)   # per-step gathers, eager
            x0c, _ = r.sample(x_T, plan, abar)   # replay of the graph captured by the first call
            eps = r.run_step(x_T, int(plan[0]), 0)
            # step API: displaced steps read what the previous call exchanged
            seq = [r.run_step(x_T, int(plan[i]), i) for i in range(steps)]
            vol = r.volumes()
            dist.barrier()   # nobody frees an exported buffer while a peer still maps it
            r.close()
            dist.barrier()
            if rank == 0:
                ref = P.PatchRunner(model, cond, h, w, mode=mode, n_devices=world,
                                    warmup_steps=warmup, dtype=dtype, device=0)
                rx0, _ = ref.sample(x_T, plan, abar)
                _, rtraj = ref.sample(x_T, plan, abar, trajectory=True)
                ref.sample(x_T, plan, abar)   # same call sequence: same byte volumes
                reps = ref.run_step(x_T, int(plan[0]), 0)
                rseq = [ref.run_step(x_T, int(plan[i]), i) for i in range(steps)]
                key = f"{mode}/w{warmup}/{dtype}"
                res[key] = {
                    "x0_equal": bool(np.array_equal(x0, rx0)),
                    "x0_replay_equal": bool(np.array_equal(x0, x0b) and np.array_equal(x0, x0c)),
                    "step_seq_equal": all(np.array_equal(a, b) for a, b in zip(seq, rseq)),
                    "traj_equal": bool(np.array_equal(traj, rtraj)),
                    "eps_equal": bool(np.array_equal(eps, reps)),
                    "x0_rel": float(np.linalg.norm(x0 - rx0) / np.linalg.norm(rx0)),
                    "finite": bool(np.isfinite(x0).all()),
                    "volumes_equal": vol == ref.volumes(),
                }
                ref.close()
            dist.barrier()
    if TRANSPORT != "ipc":
        if rank == 0:
            with open(out_path, "w") as f:
                json.dump(res, f, indent=1)
        dist.destroy_process_group()
        return
    # bad blob: wrong rank order is rejected with the reference's error class
    r = P.PatchRunner(model, cond, h, w, mode="displaced", n_devices=world, warmup_steps=1,
                      world=world, rank=rank, device=0, transport="ipc")
    try:   # a step before the handles are exchanged
        r.run_step(x_T, int(plan[0]), 0)
        res_nc = "accepted"
    except P.RuntimeFailure as e:
        res_nc = "RuntimeFailure: " + str(e)
    mine = r.ipc_handles()
    allb = [None] * world
    dist.all_gather_object(allb, mine)
    try:
        r.ipc_connect(list(reversed(allb)))
        res_bad = "accepted"
    except P.InvalidArgument as e:
        res_bad = "InvalidArgument: " + str(e)
    try:
        P.PatchRunner(model, cond, h, w, mode="displaced", n_devices=world, world=world,
                      rank=rank, device=0, transport="bogus")
        res_tp = "accepted"
    except P.InvalidArgument as e:
        res_tp = "InvalidArgument: " + str(e)
    dist.barrier()
    r.close()
    dist.barrier()
    if rank == 0:
        res["bad_blob"] = res_bad
        res["not_connected"] = res_nc
        res["bad_transport"] = res_tp
        with open(out_path, "w") as f:
            json.dump(res, f, indent=1)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

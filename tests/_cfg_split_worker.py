"""Worker of tests/test_ipc_gpu.py::test_cfg_batch_split: classifier-free guidance split across
two process groups (beyond the reference API).  Ranks [0, G) run the conditional
pass of bands 0..G-1, ranks [G, 2G) the unconditional pass of the same bands; inside a group the
bands exchange over the copy-engine (CUDA IPC) transport, and rank r swaps eps bands with rank
r +- G over a CUDA IPC pair link (argv[2] == "nccl": NCCL band transport and a two-rank NCCL
pair communicator instead).  All processes share cuda:0 (one GPU per box).  Rank 0
repeats the run with one in-process CFG runner (both passes, G bands in this process) and
writes the comparison to argv[1]: the split must be bitwise identical to it, on both halves."""
import json
import os
import sys

TRANSPORT = sys.argv[2] if len(sys.argv) > 2 else "ipc"
if TRANSPORT == "nccl":   # ranks sharing the one GPU: see _ipc_worker.py
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
    G = world // 2
    torch.cuda.set_device(0)
    groups = [dist.new_group(list(range(k * G, (k + 1) * G))) for k in range(2)]
    role, band = rank // G, rank % G
    partner = (rank + G) % world
    cfg = P.ModelConfig()
    h = w = 32
    steps = 6
    scale = 3.5
    model = P.build_model(cfg, 42)
    cond = P.random_condition(cfg.cond_dim, 7)
    uncond = 0.25 * P.random_condition(cfg.cond_dim, 8)
    x_T = P.random_normal(1, cfg.in_channels, h, w, 1234)
    abar = P.make_schedule(1000)
    plan = P.make_plan(1000, steps)
    res = {}
    cases = [("displaced", 1, "bf16"), ("displaced", 0, "fp32"), ("sync-pp", 0, "bf16")]
    if G == 1:
        cases.append(("reference", 0, "bf16"))
    for mode, warmup, dtype in cases:
        kw = dict(mode=mode, n_devices=G, warmup_steps=warmup, dtype=dtype, device=0,
                  cfg_scale=scale, uncond=uncond, cfg_pair_role=role, cfg_pair_transport=TRANSPORT)
        if G > 1:
            kw.update(world=G, rank=band, transport=TRANSPORT)
        if TRANSPORT == "nccl":
            # one communicator per group (the bands) and one per pair (the eps swap)
            ids = [[P.nccl_unique_id() for _ in range(2 + G)] if rank == 0 else None]
            dist.broadcast_object_list(ids, 0)
            kw["cfg_nccl_id"] = ids[0][2 + band]
            if G > 1:
                kw["nccl_id"] = ids[0][role]
        r = P.PatchRunner(model, cond, h, w, **kw)
        if TRANSPORT == "ipc":
            if G > 1:
                r.connect_ipc(group=groups[role])
            r.connect_pair(partner)
        x0, _ = r.sample(x_T, plan, abar)
        x0b, traj = r.sample(x_T, plan, abar, trajectory=True)   # eager
        x0c, _ = r.sample(x_T, plan, abar)   # graph replay
        eps = r.run_step(x_T, int(plan[0]), 0)
        got = [None] * world
        dist.all_gather_object(got, (x0, x0b, traj, eps, x0c))
        dist.barrier()   # nobody frees an exported buffer while a peer still maps it
        r.close()
        dist.barrier()
        if rank == 0:
            ref = P.PatchRunner(model, cond, h, w, mode=mode, n_devices=G, warmup_steps=warmup,
                                dtype=dtype, device=0, cfg_scale=scale, uncond=uncond)
            rx0, _ = ref.sample(x_T, plan, abar)
            _, rtraj = ref.sample(x_T, plan, abar, trajectory=True)
            reps = ref.run_step(x_T, int(plan[0]), 0)
            plain = P.PatchRunner(model, cond, h, w, mode=mode, n_devices=G, warmup_steps=warmup,
                                  dtype=dtype, device=0)
            px0, _ = plain.sample(x_T, plan, abar)
            ref.close()
            plain.close()
            res[f"{mode}/w{warmup}/{dtype}"] = {
                "x0_equal": all(np.array_equal(g[0], rx0) for g in got),
                "x0_replay_equal": all(np.array_equal(g[1], rx0) and np.array_equal(g[4], rx0)
                                       for g in got),
                "traj_equal": all(np.array_equal(g[2], rtraj) for g in got),
                "eps_equal": all(np.array_equal(g[3], reps) for g in got),
                "finite": bool(np.isfinite(rx0).all()),
                # guidance changes the result (the split is not silently unguided)
                "guided_rel": float(np.linalg.norm(rx0 - px0) / np.linalg.norm(px0)),
            }
        dist.barrier()
    if TRANSPORT != "ipc":
        if rank == 0:
            with open(out_path, "w") as f:
                json.dump(res, f, indent=1)
        dist.destroy_process_group()
        return
    # misuse: a blob from the wrong rank (own role), a split without a scale
    r = P.PatchRunner(model, cond, h, w, mode="reference", device=0, cfg_scale=scale,
                      cfg_pair_role=role, cfg_pair_transport="ipc")
    try:
        r.run_step(x_T, int(plan[0]), 0)
        res_nc = "accepted"
    except P.RuntimeFailure as e:
        res_nc = "RuntimeFailure: " + str(e)
    try:
        r.pair_connect(r.pair_handles())
        res_bad = "accepted"
    except P.InvalidArgument as e:
        res_bad = "InvalidArgument: " + str(e)
    try:
        P.PatchRunner(model, cond, h, w, mode="reference", device=0, cfg_pair_role=role,
                      cfg_pair_transport="ipc")
        res_ns = "accepted"
    except P.InvalidArgument as e:
        res_ns = "InvalidArgument: " + str(e)
    r.close()
    dist.barrier()
    if rank == 0:
        res["not_connected"] = res_nc
        res["bad_blob"] = res_bad
        res["no_scale"] = res_ns
        with open(out_path, "w") as f:
            json.dump(res, f, indent=1)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

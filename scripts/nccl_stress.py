"""Repeat NCCL-transport runs (two ranks on one GPU, see nccl_probe.py) and count results that
differ from the in-process run: usage nccl_stress.py REPS [MODE WARMUP DTYPE]."""
import os
import sys

rank = int(os.environ["RANK"])
os.environ["NCCL_HOSTID"] = f"pp-stress-host-{rank}"
os.environ.setdefault("NCCL_SOCKET_IFNAME", "lo")
os.environ.setdefault("NCCL_IB_DISABLE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2402_19481_b200 import patchsim as P  # noqa: E402

reps = int(sys.argv[1])
mode = sys.argv[2] if len(sys.argv) > 2 else "displaced"
warmup = int(sys.argv[3]) if len(sys.argv) > 3 else 0
dtype = sys.argv[4] if len(sys.argv) > 4 else "fp32"
from paper_2402_19481_b200 import _native as NAT  # noqa: E402
NAT.lib().pp_set_pdl(int(os.environ.get("PDL", "1")))
dist.init_process_group("gloo")
world = dist.get_world_size()
torch.cuda.set_device(0)
cfg = P.ModelConfig()
model = P.build_model(cfg, 42)
cond = P.random_condition(cfg.cond_dim, 7)
x_T = P.random_normal(1, cfg.in_channels, 32, 32, 1234)
abar, plan = P.make_schedule(1000), P.make_plan(1000, 6)
rx0 = rtraj = None
if rank == 0:
    ref = P.PatchRunner(model, cond, 32, 32, mode=mode, n_devices=world, warmup_steps=warmup,
                        dtype=dtype, device=0)
    rx0, rtraj = ref.sample(x_T, plan, abar, trajectory=True)
    reps0 = ref.run_step(x_T, int(plan[0]), 0)
    ref.close()
bad = 0
for k in range(reps):
    tp = os.environ.get("TRANSPORT", "nccl")
    kw = {}
    if tp == "nccl":
        ids = [P.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(ids, 0)
        kw["nccl_id"] = ids[0]
    r = P.PatchRunner(model, cond, 32, 32, mode=mode, n_devices=world, warmup_steps=warmup,
                      dtype=dtype, world=world, rank=rank, device=0, transport=tp, **kw)
    if tp == "ipc":
        r.connect_ipc()
    x0, traj = r.sample(x_T, plan, abar, trajectory=True)
    eps0 = r.run_step(x_T, int(plan[0]), 0)
    if rank == 0 and not np.array_equal(eps0, reps0):
        print(f"rep {k}: first run_step eps differs (max {float(np.abs(eps0 - reps0).max()):.3e})", flush=True)
    both = [None] * world
    dist.all_gather_object(both, (x0, traj))
    if rank == 0 and not np.array_equal(x0, rx0):
        same = [bool(np.array_equal(both[0][1][i], both[1][1][i])) for i in range(len(plan))]
        steps = [bool(np.array_equal(traj[i], rtraj[i])) for i in range(len(plan))]
        rows = [np.unique(np.nonzero(traj[i] - rtraj[i])[2]).tolist() for i in range(len(plan))]
        print(f"   per-step equal {steps}; rank0==rank1 traj {same}, x0 {np.array_equal(both[0][0], both[1][0])}; "
              f"rows step1 {rows[1][:8]}..{len(rows[1])} step2 {len(rows[2])}", flush=True)
        bad += 1
        first = next(i for i in range(len(plan)) if not np.array_equal(traj[i], rtraj[i])) \
            if not np.array_equal(traj, rtraj) else -1
        print(f"rep {k}: x0 differs (max {float(np.abs(x0 - rx0).max()):.3e}), first differing "
              f"trajectory step {first}", flush=True)
    dist.barrier()
    r.close()
    dist.barrier()
if rank == 0:
    print(f"{mode} w{warmup} {dtype}: {bad} of {reps} runs differ", flush=True)
dist.destroy_process_group()

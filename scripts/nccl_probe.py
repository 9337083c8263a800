"""Probe: NCCL transport with two ranks on ONE GPU.  NCCL refuses two ranks of one host on one
device ("Duplicate GPU"); giving each rank its own NCCL_HOSTID makes them look like two hosts,
so NCCL connects them over its socket transport (loopback) -- slow, but the runtime's NCCL
transport code (send/recv pairs, all-gathers, graph capture) runs for real."""
import os
import sys

rank = int(os.environ["RANK"])
os.environ["NCCL_HOSTID"] = f"pp-probe-host-{rank}"
os.environ.setdefault("NCCL_SOCKET_IFNAME", "lo")
os.environ.setdefault("NCCL_IB_DISABLE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2402_19481_b200 import patchsim as P  # noqa: E402

dist.init_process_group("gloo")
world = dist.get_world_size()
torch.cuda.set_device(0)
cfg = P.ModelConfig()
model = P.build_model(cfg, 42)
cond = P.random_condition(cfg.cond_dim, 7)
x_T = P.random_normal(1, cfg.in_channels, 32, 32, 1234)
abar, plan = P.make_schedule(1000), P.make_plan(1000, 6)
ids = [P.nccl_unique_id() if rank == 0 else None]
dist.broadcast_object_list(ids, 0)
r = P.PatchRunner(model, cond, 32, 32, mode="displaced", n_devices=world, warmup_steps=1,
                  world=world, rank=rank, device=0, transport="nccl", nccl_id=ids[0])
x0, _ = r.sample(x_T, plan, abar)
x0b, _ = r.sample(x_T, plan, abar)
print(f"rank {rank}: sample ok", flush=True)
dist.barrier()
if rank == 0:
    ref = P.PatchRunner(model, cond, 32, 32, mode="displaced", n_devices=world, warmup_steps=1, device=0)
    rx0, _ = ref.sample(x_T, plan, abar)
    print("x0 equal", np.array_equal(x0, rx0), "replay equal", np.array_equal(x0, x0b),
          "rel", float(np.linalg.norm(x0 - rx0) / np.linalg.norm(rx0)), flush=True)
r.close()
dist.barrier()
dist.destroy_process_group()

"""Does NCCL itself deliver correct data with two ranks on one GPU under distinct NCCL_HOSTIDs?
Fresh communicators, the runtime's op mix (send/recv pairs + in-place all-gathers in one group)."""
import os
import sys

rank = int(os.environ["RANK"])
os.environ["NCCL_HOSTID"] = f"pp-self-host-{rank}"
os.environ.setdefault("NCCL_SOCKET_IFNAME", "lo")
os.environ.setdefault("NCCL_IB_DISABLE", "1")
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

dist.init_process_group("gloo")
torch.cuda.set_device(0)
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
bad = 0
for k in range(reps):
    pg = dist.new_group([0, 1], backend="nccl")
    g = torch.Generator(device="cpu").manual_seed(k)
    for it in range(5):
        n = 4096 * (it + 1)
        mine = torch.randn(2, n, generator=g)[rank].cuda()
        buf = torch.empty(2 * n, device="cuda")
        buf[rank * n:(rank + 1) * n] = mine
        out = torch.empty(n, device="cuda")
        peer = 1 - rank
        with dist._coalescing_manager(group=pg):
            dist.all_gather_into_tensor(buf, buf[rank * n:(rank + 1) * n].clone(), group=pg)
        ops = [dist.P2POp(dist.isend, mine, peer, pg), dist.P2POp(dist.irecv, out, peer, pg)]
        for r in dist.batch_isend_irecv(ops):
            r.wait()
        torch.cuda.synchronize()
        ref = torch.randn(2, n, generator=torch.Generator().manual_seed(k))
        # regenerate the peer's data with the same generator sequence
        gg = torch.Generator(device="cpu").manual_seed(k)
        for j in range(it + 1):
            full = torch.randn(2, 4096 * (j + 1), generator=gg)
        ok = torch.equal(buf.cpu(), full.reshape(-1)) and torch.equal(out.cpu(), full[peer])
        if not ok:
            bad += 1
            print(f"rank {rank} rep {k} it {it}: WRONG", flush=True)
    dist.destroy_process_group(pg)
print(f"rank {rank}: {bad} wrong of {reps * 5}", flush=True)
dist.destroy_process_group()

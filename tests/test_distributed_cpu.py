"""Multi-process (one rank per GPU) host logic, exercised on CPU with gloo, world size 2.

Covers what the NCCL layout runs on the host: the ncclUniqueId rendezvous through
torch.distributed, the rank -> row-band mapping (partition_rows / derive_patch_spec must
agree across ranks), the rank-ordered stitching of gathered bands (pp_assemble_bands, the
eps / x0 stitch of run_workers, proj/src/runtime.cpp:368-377), the per-rank MAC split
(total / N, proj/tests/test_runtime.cpp:355-369) and bench.py's max-over-ranks timing.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import ctypes as C
        from paper_2402_19481_b200 import _native as N
        from paper_2402_19481_b200 import patchsim as P
        # (1) ncclUniqueId rendezvous exactly as bench.py does it
        try:
            uid = P.nccl_unique_id() if rank == 0 else None
        except Exception:
            uid = bytes(range(128)) if rank == 0 else None   # no NCCL bootstrap NIC here
        obj = [uid]
        dist.broadcast_object_list(obj, src=0)
        ids = [None] * world
        dist.all_gather_object(ids, obj[0])
        assert len(ids[0]) == 128 and ids[0] == ids[1]
        # (2) rank -> band mapping agrees on every rank and tiles the image
        H = W = 32
        cfg = P.ModelConfig()
        m = P.build_model(cfg, 42)
        bands = P.partition_rows(H, world, W)
        mine = bands[rank]
        lin, lout = m.patch_spec(mine)
        allspec = [None] * world
        dist.all_gather_object(allspec, (mine, lin.tolist(), lout.tolist()))
        assert [s[0] for s in allspec] == bands
        for layer in range(lin.shape[0]):
            rows = sorted((s[1][layer][0], s[1][layer][1]) for s in allspec)
            assert rows[0][0] == 0 and rows[-1][1] == allspec[0][1][layer][2]
            assert all(rows[i][1] == rows[i + 1][0] for i in range(world - 1))
        # (3) each rank owns its band of a global image; gather + stitch in rank order
        img = np.arange(4 * H * W, dtype=np.float32).reshape(4, H, W)
        band = np.ascontiguousarray(img[:, mine[0]:mine[1], :])
        t = torch.from_numpy(band.reshape(-1))
        parts = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(parts, t)
        gathered = torch.cat(parts).numpy()
        out = np.zeros_like(img)
        N.check(N.lib().pp_assemble_bands(gathered.ctypes.data_as(C.c_void_p), world, 4,
                                          H // world, W, out.ctypes.data_as(C.c_void_p)))
        assert np.array_equal(out, img)
        # (4) per-rank MACs are exactly total / N
        macs = sum(m.macs_of_layer(layer, tuple(int(v) for v in lin[layer]))
                   for layer in range(lin.shape[0]))
        tot = torch.tensor([macs], dtype=torch.float64)
        dist.all_reduce(tot)
        assert int(tot.item()) == m.total_macs(H, W) and macs * world == m.total_macs(H, W)
        # (5) bench.py's timing reduction: the job time is the max over ranks
        mytime = torch.tensor([1.0 + rank], dtype=torch.float64)
        dist.all_reduce(mytime, op=dist.ReduceOp.MAX)
        assert mytime.item() == float(world)
        q.put((rank, "ok"))
    except Exception as e:  # surface the failure to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_two_rank_host_logic():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert results == {0: "ok", 1: "ok"}, results

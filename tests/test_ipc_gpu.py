"""Multi-process transports: the copy-engine transport (CUDA IPC peer mappings + stream memory
operations) and the NCCL transport.  A world-2 / world-4 run, one process
per band, must be bitwise identical to the in-process multi-band run (same kernels, same data;
only the exchange mechanism differs) in every mode, dtype, with and without trajectories, for
graph capture and replay, and through the step API.  The box has one GPU: all ranks share it
(NCCL under a per-rank NCCL_HOSTID, see _ipc_worker.py)."""
import json
import os
import signal
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(cmd, what):
    """Run a torchrun command in its own session; on a hang kill it AND its workers (exact
    PIDs: the workers may sit in sessions of their own and keep the output pipe open)."""
    import psutil
    p = subprocess.Popen(cmd, cwd=ROOT, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True,
                         start_new_session=True)
    try:
        log, _ = p.communicate(timeout=300)
    except subprocess.TimeoutExpired:
        procs = [p.pid] + [c.pid for c in psutil.Process(p.pid).children(recursive=True)]
        for pid in procs:
            try:
                os.kill(pid, signal.SIGKILL)
            except ProcessLookupError:
                pass
        log, _ = p.communicate(timeout=60)
        pytest.fail(f"{what} timed out:\n" + log[-3000:])
    assert p.returncode == 0, log[-5000:]


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.gpu
@pytest.mark.parametrize("transport", ["ipc", "nccl"])
@pytest.mark.parametrize("world", [2, 4])
def test_transport_matches_inprocess(tmp_path, world, transport):
    # world 4: interior bands exchange halos with both neighbours.  NCCL: every rank on the one
    # GPU under its own NCCL_HOSTID (NCCL's socket transport over loopback; _ipc_worker.py)
    out = tmp_path / "x.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "tests", "_ipc_worker.py"), str(out), transport]
    _run(cmd, f"{transport} world-{world} run")
    res = json.loads(out.read_text())
    assert len([k for k in res if "/" in k]) == 6
    for key in [k for k in res if "/" in k]:
        r = res[key]
        assert r["finite"], key
        assert r["x0_equal"] and r["traj_equal"] and r["eps_equal"], (key, r)
        assert r["x0_replay_equal"], (key, r)   # graph capture, replay and eager agree
        assert r["step_seq_equal"], (key, r)
        assert r["volumes_equal"], (key, r)
    if transport != "ipc":
        return
    assert res["bad_blob"].startswith("InvalidArgument"), res["bad_blob"]
    assert res["bad_transport"].startswith("InvalidArgument"), res["bad_transport"]
    assert res["not_connected"].startswith("RuntimeFailure") and "not connected" in res["not_connected"]


@pytest.mark.gpu
@pytest.mark.parametrize("transport", ["ipc", "nccl"])
@pytest.mark.parametrize("world", [2, 4])
def test_cfg_batch_split(tmp_path, world, transport):
    # classifier-free guidance split across two groups of world/2 ranks (conditional /
    # unconditional pass), eps swapped over a CUDA IPC pair link: both halves must equal the
    # in-process CFG runner bit for bit
    out = tmp_path / "cfg.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "tests", "_cfg_split_worker.py"), str(out), transport]
    _run(cmd, f"CFG split {transport} world-{world} run")
    res = json.loads(out.read_text())
    keys = [k for k in res if "/" in k]
    assert len(keys) >= 3
    for key in keys:
        r = res[key]
        assert r["finite"], key
        assert r["x0_equal"] and r["x0_replay_equal"] and r["traj_equal"] and r["eps_equal"], (key, r)
        assert r["guided_rel"] > 1e-3, (key, r)
    if transport != "ipc":
        return
    assert res["not_connected"].startswith("RuntimeFailure") and "not connected" in res["not_connected"]
    assert res["bad_blob"].startswith("InvalidArgument"), res["bad_blob"]
    assert res["no_scale"].startswith("InvalidArgument"), res["no_scale"]

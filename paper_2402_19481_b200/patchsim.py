"""Python mirror of the reference's public interface for the hot path.

Same names, argument meaning and error behaviour as ``patchsim`` (the reference
C++ library, ``proj/include/patchsim/*.hpp``), backed by the C ABI of
``libpp_b200.so``.  Tensors are numpy float32 arrays in NCHW, like
``patchsim::Tensor``.  Errors: ``InvalidArgument`` (std::invalid_argument) and
``RuntimeFailure`` (std::runtime_error) carry the reference's message text.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N
from ._native import CudaError, InvalidArgument, NcclError, RuntimeFailure  # noqa: F401

KINDS = ["Conv", "GroupNorm", "SiLU", "DownConv", "Upsample", "SelfAttn", "CrossAttn", "Linear",
         "AddSkip", "AddTimeEmb"]


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


@dataclass
class ModelConfig:
    """proj/include/patchsim/model.hpp:30-41."""
    in_channels: int = 4
    base_channels: int = 16
    levels: int = 3
    groups: int = 4
    cond_dim: int = 8
    attn_at_level: int = -1
    # deeper graphs (beyond the reference API; defaults = the reference graph)
    res_blocks: int = 1
    attn_levels: int = 0
    attn_depth: int = 1
    attn_up: int = 0

    def c(self):
        return N.ModelConfig(self.in_channels, self.base_channels, self.levels, self.groups,
                             self.cond_dim, self.attn_at_level, self.res_blocks, self.attn_levels,
                             self.attn_depth, self.attn_up)

    def depth_divisor(self):
        return 1 << (self.levels - 1)


SDXL_SHAPE = ModelConfig(4, 320, 3, 32, 2048, -1)


class Model:
    """build_model / Model (proj/src/model.cpp:179-218); weights live on the host until a
    runner uploads them."""

    def __init__(self, handle, cfg):
        self._h = handle
        self.cfg = cfg

    @classmethod
    def build(cls, cfg: ModelConfig, seed: int):
        h = C.c_void_p()
        c = cfg.c()
        N.check(N.lib().pp_model_build(C.byref(c), seed, C.byref(h)))
        return cls(h, cfg)

    @classmethod
    def from_pool(cls, cfg: ModelConfig, weights):
        """Graph of cfg with a caller weight pool (dump_weights order)."""
        pool = _f32(np.concatenate([np.asarray(w, dtype=np.float32).reshape(-1) for w in weights]))
        h = C.c_void_p()
        c = cfg.c()
        N.check(N.lib().pp_model_from_pool(C.byref(c), _p(pool), pool.size, C.byref(h)))
        return cls(h, cfg)

    def __del__(self):
        # (module globals may already be None at interpreter shutdown)
        if getattr(self, "_h", None) and N is not None and N._lib is not None:
            N._lib.pp_model_destroy(self._h)
            self._h = None

    @property
    def layers(self):
        out = []
        for i in range(N.lib().pp_model_num_layers(self._h)):
            d = N.LayerDesc()
            N.check(N.lib().pp_model_layer(self._h, i, C.byref(d)))
            dd = {f: getattr(d, f) for f, _ in N.LayerDesc._fields_}
            dd["kind"] = KINDS[dd["kind"]]
            out.append(dd)
        return out

    def weights(self):
        ws = []
        for i in range(N.lib().pp_model_num_weights(self._h)):
            s = np.zeros(4, dtype=np.int32)
            N.check(N.lib().pp_model_weight_shape(self._h, i, _p(s)))
            ws.append(tuple(int(v) for v in s))
        pool = np.zeros(N.lib().pp_model_pool_size(self._h), dtype=np.float32)
        N.check(N.lib().pp_model_pool(self._h, _p(pool)))
        out, off = [], 0
        for s in ws:
            n = int(np.prod(s))
            out.append(pool[off:off + n].reshape(s))
            off += n
        return out

    def zero_weights(self, keep_biases: bool):
        N.check(N.lib().pp_model_zero_weights(self._h, int(keep_biases)))

    def total_macs(self, h, w):
        return int(N.lib().pp_model_total_macs(self._h, h, w))

    def macs_of_layer(self, layer, region):
        r = np.array(region, dtype=np.int32)
        return int(N.lib().pp_macs_of_layer(self._h, layer, _p(r)))

    def patch_spec(self, region):
        L = N.lib().pp_model_num_layers(self._h)
        r = np.array(region, dtype=np.int32)
        a = np.zeros(4 * L, dtype=np.int32)
        b = np.zeros(4 * L, dtype=np.int32)
        N.check(N.lib().pp_derive_patch_spec(self._h, _p(r), _p(a), _p(b)))
        return a.reshape(L, 4), b.reshape(L, 4)


def build_model(cfg: ModelConfig, seed: int) -> Model:
    return Model.build(cfg, seed)


def partition_rows(h, n_devices, full_w):
    out = np.zeros(4 * max(n_devices, 1), dtype=np.int32)
    N.check(N.lib().pp_partition_rows(h, n_devices, full_w, _p(out)))
    return [tuple(int(v) for v in out[4 * i:4 * i + 4]) for i in range(n_devices)]


def derive_patch_spec(model: Model, region):
    return model.patch_spec(region)


def corrected_gn_stats(fresh, prev_local, prev_global):
    g = len(fresh[0])
    arr = [np.ascontiguousarray(np.concatenate(s), dtype=np.float64)
           for s in (fresh, prev_local, prev_global)]
    if not (len(arr[0]) == len(arr[1]) == len(arr[2])):
        raise InvalidArgument("corrected_gn_stats: group-count mismatch")
    out = np.zeros(2 * g)
    N.check(N.lib().pp_corrected_gn_stats(g, _p(arr[0]), _p(arr[1]), _p(arr[2]), _p(out)))
    return out[:g], out[g:]


def make_schedule(total=1000, beta_start=1e-4, beta_end=2e-2):
    out = np.zeros(total)
    N.check(N.lib().pp_make_schedule(total, beta_start, beta_end, _p(out)))
    return out


def make_plan(total, num_steps):
    out = np.zeros(num_steps, dtype=np.int32)
    N.check(N.lib().pp_make_plan(total, num_steps, _p(out)))
    return [int(v) for v in out]


def random_normal(n, c, h, w, seed):
    out = np.zeros((n, c, h, w), dtype=np.float32)
    N.check(N.lib().pp_random_normal(n, c, h, w, seed, _p(out)))
    return out


def random_condition(dim, seed):
    out = np.zeros(dim, dtype=np.float32)
    N.check(N.lib().pp_random_condition(dim, seed, _p(out)))
    return out


@dataclass
class RunnerOptions:
    """proj/include/patchsim/runtime.hpp:47-54, plus the B200 placement/precision knobs."""
    mode: str = "reference"
    n_devices: int = 1
    warmup_steps: int = 4
    gn_scheme: str = "corrected"
    dtype: str = "bf16"
    world: int = 1
    rank: int = 0
    nccl_id: bytes | None = None
    device: int = 0
    profile: bool = False
    transport: str = "nccl"          # world > 1: "nccl" or "ipc" (CUDA IPC + copy engines)
    no_comm: bool = False            # ablation only ("No Comm."): exchanges skipped
    stress: bool = False             # --stress-sched: scheduling noise (results unchanged)
    stress_seed: int = 0xC0FFEE
    cfg_scale: float = 0.0           # classifier-free guidance (beyond the reference API)
    uncond: object = None            # unconditional condition (cond_dim floats; None = zeros)
    cfg_nccl_id: bytes | None = None # world > 1 + NCCL: the unconditional pass's unique id;
                                     # batch split + NCCL: the pair communicator's unique id
    cfg_pair_role: int = -1          # CFG batch split: 0 conditional / 1 unconditional rank
    cfg_pair_transport: str = "nccl" # batch split eps swap: "nccl" or "ipc"


class PatchRunner:
    """PatchRunner (proj/include/patchsim/runtime.hpp:57-108) on B200 bands."""

    def __init__(self, model: Model, cond, h, w, opts: RunnerOptions | None = None, **kw):
        opts = opts or RunnerOptions(**kw)
        self.opts = opts
        self.model = model
        self.h, self.w = h, w
        # a 2-D cond [T][cond_dim] is T condition tokens (multi-token cross-attention, beyond
        # the reference API); 1-D is the reference's single condition vector
        tokens = int(np.asarray(cond).shape[0]) if np.asarray(cond).ndim == 2 else 1
        cond = _f32(cond)
        o = N.RunnerOpts()
        N.lib().pp_runner_opts_default(C.byref(o))
        o.mode = N.MODES[opts.mode]
        o.n_devices = opts.n_devices
        o.warmup_steps = opts.warmup_steps
        o.gn_scheme = N.GN_SCHEMES[opts.gn_scheme]
        o.dtype = N.DTYPES[opts.dtype]
        o.world = opts.world
        o.rank = opts.rank
        self._id = C.create_string_buffer(bytes(opts.nccl_id), 128) if opts.nccl_id else None
        o.nccl_id = C.cast(self._id, C.c_void_p) if self._id is not None else None
        o.device = opts.device
        o.profile = int(opts.profile)
        if opts.transport not in N.TRANSPORTS:
            raise InvalidArgument(f"unknown transport '{opts.transport}'")
        o.transport = N.TRANSPORTS[opts.transport]
        o.no_comm = int(opts.no_comm)
        o.stress = int(opts.stress)
        o.stress_seed = int(opts.stress_seed)
        o.cfg_scale = float(opts.cfg_scale)
        o.cond_tokens = tokens
        if opts.uncond is not None:
            self._uncond = _f32(opts.uncond)
            if self._uncond.size != cond.size:
                raise InvalidArgument(f"classifier-free guidance: uncond length {self._uncond.size} "
                                      f"!= condition length {cond.size}")
            o.uncond = self._uncond.ctypes.data
        o.cfg_pair_role = int(opts.cfg_pair_role)
        if opts.cfg_pair_transport not in N.TRANSPORTS:
            raise InvalidArgument(f"unknown transport '{opts.cfg_pair_transport}'")
        o.cfg_pair_transport = N.TRANSPORTS[opts.cfg_pair_transport]
        if opts.cfg_nccl_id is not None:
            self._cfg_id = C.create_string_buffer(bytes(opts.cfg_nccl_id), 128)
            o.cfg_nccl_id = C.cast(self._cfg_id, C.c_void_p)
        h_ = C.c_void_p()
        N.check(N.lib().pp_runner_create(model._h, _p(cond), cond.size, h, w, C.byref(o),
                                         C.byref(h_)))
        self._r = h_
        self.n_devices = 1 if opts.mode == "reference" else opts.n_devices

    def ipc_handles(self) -> bytes:
        """This rank's CUDA IPC handle blob (transport "ipc"), to be all-gathered."""
        n = C.c_long()
        N.check(N.lib().pp_runner_ipc_export(self._r, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value)
        N.check(N.lib().pp_runner_ipc_export(self._r, buf, n.value, C.byref(n)))
        return buf.raw

    def ipc_connect(self, blobs) -> None:
        """Open every rank's receive buffers (blobs in rank order)."""
        blobs = [bytes(b) for b in blobs]
        if len({len(b) for b in blobs}) != 1:
            raise InvalidArgument("ipc_connect: blobs differ in size")
        flat = C.create_string_buffer(b"".join(blobs), len(blobs) * len(blobs[0]))
        N.check(N.lib().pp_runner_ipc_connect(self._r, flat, len(blobs[0])))

    def connect_ipc(self, group=None) -> None:
        """all-gather the handle blobs over torch.distributed (any backend) and connect."""
        import torch.distributed as dist
        mine = self.ipc_handles()
        allb = [None] * dist.get_world_size(group)
        dist.all_gather_object(allb, mine, group=group)
        self.ipc_connect(allb)

    def pair_handles(self) -> bytes:
        """CFG batch split over CUDA IPC: this rank's pair-link handle blob."""
        n = C.c_long()
        N.check(N.lib().pp_runner_pair_export(self._r, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value)
        N.check(N.lib().pp_runner_pair_export(self._r, buf, n.value, C.byref(n)))
        return buf.raw

    def pair_connect(self, blob) -> None:
        """Open the partner rank's pair-link receive buffers."""
        blob = bytes(blob)
        buf = C.create_string_buffer(blob, len(blob))
        N.check(N.lib().pp_runner_pair_connect(self._r, buf, len(blob)))

    def connect_pair(self, partner: int, group=None) -> None:
        """all-gather the pair blobs over torch.distributed and connect to `partner` (its rank
        in `group`)."""
        import torch.distributed as dist
        mine = self.pair_handles()
        allb = [None] * dist.get_world_size(group)
        dist.all_gather_object(allb, mine, group=group)
        self.pair_connect(allb[partner])

    def close(self):
        if getattr(self, "_r", None) and N is not None and N._lib is not None:
            N._lib.pp_runner_destroy(self._r)
            self._r = None

    def __del__(self):
        self.close()

    def _step(self, entry, x, t, step_index):
        x = _f32(x)
        eps = np.zeros_like(x)
        N.check(N.lib().pp_runner_step(self._r, N.ENTRIES[entry], _p(x), t, step_index, _p(eps)))
        return eps

    def run_step(self, x, t, step_index):
        return self._step("run_step", x, t, step_index)

    def step_reference(self, x, t, step_index):
        return self._step("reference", x, t, step_index)

    def step_naive(self, x, t, step_index):
        return self._step("naive", x, t, step_index)

    def step_sync(self, x, t, step_index):
        return self._step("sync", x, t, step_index)

    def step_displaced(self, x, t, step_index):
        return self._step("displaced", x, t, step_index)

    def patch_spec(self, device):
        L = N.lib().pp_model_num_layers(self.model._h)
        a = np.zeros(4 * L, dtype=np.int32)
        b = np.zeros(4 * L, dtype=np.int32)
        N.check(N.lib().pp_runner_patch_spec(self._r, device, _p(a), _p(b)))
        return a.reshape(L, 4), b.reshape(L, 4)

    def cached_input(self, device, layer):
        s = np.zeros(4, dtype=np.int32)
        n = N.lib().pp_runner_cached_input(self._r, device, layer, None, _p(s))
        if n < 0:
            N.check(N.PP_EINVAL)
        if n == 0:
            return None
        a = np.zeros(tuple(int(v) for v in s), dtype=np.float32)
        N.lib().pp_runner_cached_input(self._r, device, layer, _p(a), _p(s))
        return a

    def total_macs(self):
        return int(N.lib().pp_runner_total_macs(self._r))

    def step_device_macs(self, step):
        out = np.zeros(self.n_devices, dtype=np.uint64)
        N.check(N.lib().pp_runner_step_device_macs(self._r, step, _p(out)))
        return [int(v) for v in out]

    def volumes(self):
        v = np.zeros(6, dtype=np.uint64)
        N.check(N.lib().pp_runner_volumes(self._r, _p(v)))
        return dict(zip(["allgather_recv", "allgather_sent", "halo_recv", "halo_sent",
                         "statreduce_recv", "statreduce_sent"], (int(x) for x in v)))

    def trace(self, device=0):
        """RawTrace events of one device (PatchRunner::trace(), trace.hpp:18-35) as tuples
        (device, step, layer, kind, prim, macs, bytes_recv, bytes_sent, tag)."""
        n = N.lib().pp_runner_trace(self._r, device, None, 0)
        if n < 0:
            N.check(-1)
        out = np.zeros((max(n, 1), 9), dtype=np.uint64)
        N.lib().pp_runner_trace(self._r, device, _p(out), n)
        rows = []
        for r in out[:n]:
            v = [int(x) for x in r]
            v[2] = v[2] - (1 << 64) if v[2] >= (1 << 63) else v[2]
            rows.append(tuple(v))
        return rows

    def sample(self, x_T, timesteps, alpha_bar, trajectory=False):
        """sample() (proj/src/sampler.cpp:76-95) with the loop on the GPU."""
        x_T = _f32(x_T)
        ts = np.ascontiguousarray(timesteps, dtype=np.int32)
        ab = np.ascontiguousarray(alpha_bar, dtype=np.float64)
        x0 = np.zeros_like(x_T)
        traj = np.zeros((len(ts),) + x_T.shape, dtype=np.float32) if trajectory else None
        N.check(N.lib().pp_runner_sample(self._r, _p(x_T), _p(ts), len(ts), _p(ab), len(ab),
                                         _p(x0), _p(traj)))
        return x0, traj

    def profile(self):
        o = np.zeros(7)
        N.check(N.lib().pp_runner_profile(self._r, _p(o)))
        return dict(zip(["conv_ms", "conv_flops", "gemm_ms", "gemm_flops", "gn_ms", "other_ms",
                         "launches"], o.tolist()))

    def launches(self):
        return int(N.lib().pp_runner_launches(self._r))

    def last_device_ms(self):
        return float(N.lib().pp_runner_last_device_ms(self._r))

    def set_profile(self, on: bool):
        N.check(N.lib().pp_runner_set_profile(self._r, int(on)))


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    N.check(N.lib().pp_nccl_unique_id(buf))
    return buf.raw


@dataclass
class RunConfig:
    """proj/include/patchsim/runtime.hpp:112-130."""
    mode: str = "reference"
    n_devices: int = 1
    h: int = 48
    w: int = 48
    num_steps: int = 50
    warmup: int = 4
    gn_scheme: str = "corrected"
    dtype: str = "bf16"
    model_seed: int = 42
    noise_seed: int = 1234
    cond_seed: int = 7
    model: ModelConfig = None
    schedule_steps: int = 1000
    beta_start: float = 1e-4
    beta_end: float = 2e-2

    def c(self):
        m = self.model or ModelConfig()
        return N.RunConfig(N.MODES[self.mode], self.n_devices, self.h, self.w, self.num_steps,
                           self.warmup, N.GN_SCHEMES[self.gn_scheme], N.DTYPES[self.dtype],
                           self.model_seed, self.noise_seed, self.cond_seed, m.c(),
                           self.schedule_steps, self.beta_start, self.beta_end)

    def validate(self):
        c = self.c()
        N.check(N.lib().pp_run_config_validate(C.byref(c)))


def run_sampling(cfg: RunConfig, trajectory=False):
    """run_sampling (proj/src/runtime.cpp:494-526): returns dict(x0, trajectory, total_macs)."""
    m = cfg.model or ModelConfig()
    c = cfg.c()
    x0 = np.zeros((1, m.in_channels, cfg.h, cfg.w), dtype=np.float32)
    traj = (np.zeros((cfg.num_steps, 1, m.in_channels, cfg.h, cfg.w), dtype=np.float32)
            if trajectory else None)
    macs = C.c_uint64()
    N.check(N.lib().pp_run_sampling(C.byref(c), _p(x0), _p(traj), C.byref(macs)))
    return {"x0": x0, "trajectory": traj, "total_macs": int(macs.value)}

"""TEST INFRASTRUCTURE ONLY: ctypes access to the reference's own CPU path.

Loads ``oracle/_ref/libpatchsim_ref.so`` -- the unmodified reference sources
(``/root/reference/proj/src/*.cpp``) compiled by ``oracle/Makefile`` together
with the C shim ``oracle/ref_capi.cpp``.  Only ``tests/``, ``__graft_entry__``
(smoke / build) and ``bench.py``'s cpu_baseline / ``--impl reference`` leg may
import this module; the product never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libpatchsim_ref.so")
REF_SRC = "/root/reference/proj"

_lib = None

# LayerKind order, proj/include/patchsim/model.hpp:15-26
KINDS = ["Conv", "GroupNorm", "SiLU", "DownConv", "Upsample", "SelfAttn",
         "CrossAttn", "Linear", "AddSkip", "AddTimeEmb"]
MODES = {"reference": 0, "naive": 1, "sync-pp": 2, "displaced": 3}
GN_SCHEMES = {"corrected": 0, "stale": 1, "separate": 2}


class RefError(Exception):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


class RefInvalidArgument(RefError, ValueError):
    pass


class RefRuntimeError(RefError, RuntimeError):
    pass


def build():
    """Compile the reference (only possible where /root/reference exists)."""
    if os.path.isdir(REF_SRC):
        subprocess.run(["make", "-s", "-C", HERE], check=True)


def available():
    return os.path.exists(LIB_PATH) or os.path.isdir(REF_SRC)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        L.ref_last_error.restype = C.c_char_p
        L.ref_model_build.restype = C.c_void_p
        L.ref_model_build.argtypes = [C.c_void_p, C.c_uint64]
        L.ref_runner_create.restype = C.c_void_p
        L.ref_runner_create.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int,
                                        C.c_int, C.c_int, C.c_int, C.c_int, C.c_int]
        for name in ["ref_model_free", "ref_runner_free"]:
            getattr(L, name).argtypes = [C.c_void_p]
        L.ref_model_total_macs.restype = C.c_uint64
        L.ref_model_total_macs.argtypes = [C.c_void_p, C.c_int, C.c_int]
        L.ref_runner_total_macs.restype = C.c_uint64
        L.ref_runner_total_macs.argtypes = [C.c_void_p]
        L.ref_runner_cached_input.restype = C.c_long
        L.ref_macs_of_layer.restype = C.c_uint64
        L.ref_macs_of_layer.argtypes = [C.c_void_p] + [C.c_int] * 5
        L.ref_run_sampling.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_double,
                                       C.c_double, C.c_void_p, C.c_void_p, C.c_void_p,
                                       C.c_void_p]
        L.ref_attention.argtypes = [C.c_void_p] * 3 + [C.c_int] * 5 + [C.c_float, C.c_void_p]
        L.ref_group_norm_apply.argtypes = ([C.c_void_p] + [C.c_int] * 7 + [C.c_void_p] * 4 +
                                           [C.c_float, C.c_void_p])
        L.ref_ddim_update.argtypes = [C.c_void_p, C.c_void_p, C.c_long, C.c_double,
                                      C.c_double, C.c_void_p]
        L.ref_silu.argtypes = [C.c_void_p, C.c_long, C.c_void_p]
        L.ref_make_schedule.argtypes = [C.c_int, C.c_double, C.c_double, C.c_void_p]
        L.ref_random_normal.argtypes = [C.c_int] * 4 + [C.c_uint64, C.c_void_p]
        L.ref_random_condition.argtypes = [C.c_int, C.c_uint64, C.c_void_p]
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def _check(rc):
    if rc == 0:
        return
    msg = lib().ref_last_error().decode()
    if rc == 1:
        raise RefInvalidArgument(rc, msg)
    raise RefRuntimeError(rc, msg)


def f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


class Model:
    """Handle to a reference ``Model`` (build_model, proj/src/model.cpp:179)."""

    def __init__(self, cfg, seed):
        self.cfg = tuple(cfg)
        c6 = np.array(self.cfg, dtype=np.int32)
        h = lib().ref_model_build(_p(c6), seed)
        if not h:
            raise RefInvalidArgument(1, lib().ref_last_error().decode())
        self.h = h
        self.seed = seed

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.ref_model_free(self.h)

    def layers(self):
        n = lib().ref_model_num_layers(C.c_void_p(self.h))
        out = []
        for i in range(n):
            v = np.zeros(15, dtype=np.int32)
            eps = C.c_float()
            lib().ref_model_layer(C.c_void_p(self.h), i, _p(v), C.byref(eps))
            d = dict(zip(["kind", "in_ch", "out_ch", "kernel", "stride", "pad", "groups",
                          "cond_dim", "skip_source", "scale_in", "scale_out", "weight",
                          "bias", "weight2", "bias2"], [int(x) for x in v]))
            d["kind"] = KINDS[d["kind"]]
            d["eps"] = eps.value
            d["id"] = i
            out.append(d)
        return out

    def weights(self):
        n = lib().ref_model_num_weights(C.c_void_p(self.h))
        ws = []
        for i in range(n):
            s = np.zeros(4, dtype=np.int32)
            lib().ref_model_weight_shape(C.c_void_p(self.h), i, _p(s))
            a = np.zeros(tuple(int(x) for x in s), dtype=np.float32)
            lib().ref_model_weight_get(C.c_void_p(self.h), i, _p(a))
            ws.append(a)
        return ws

    def set_weight(self, i, arr):
        a = f32(arr)
        lib().ref_model_weight_set(C.c_void_p(self.h), i, _p(a))

    def zero_weights(self, keep_biases):
        lib().ref_model_zero_weights(C.c_void_p(self.h), int(keep_biases))

    def total_macs(self, h, w):
        return int(lib().ref_model_total_macs(C.c_void_p(self.h), h, w))

    def macs_of_layer(self, layer, r0, r1, fh, fw):
        return int(lib().ref_macs_of_layer(C.c_void_p(self.h), layer, r0, r1, fh, fw))

    def forward_collect(self, x, t, cond):
        x = f32(x)
        _, c, h, w = x.shape
        shapes = [(1, d["out_ch"], h // d["scale_out"], w // d["scale_out"])
                  for d in self.layers()]
        total = sum(int(np.prod(s)) for s in shapes)
        buf = np.zeros(total, dtype=np.float32)
        cond = f32(cond)
        _check(lib().ref_forward_collect(C.c_void_p(self.h), _p(x), c, h, w, t, _p(cond),
                                         len(cond), _p(buf)))
        outs, off = [], 0
        for s in shapes:
            n = int(np.prod(s))
            outs.append(buf[off:off + n].reshape(s))
            off += n
        return outs

    def forward_full(self, x, t, cond):
        x = f32(x)
        out = np.zeros_like(x)
        cond = f32(cond)
        _check(lib().ref_forward_full(C.c_void_p(self.h), _p(x), x.shape[1], x.shape[2],
                                      x.shape[3], t, _p(cond), len(cond), _p(out)))
        return out

    def patch_spec(self, region):
        L = lib().ref_model_num_layers(C.c_void_p(self.h))
        r = np.array(region, dtype=np.int32)
        out = np.zeros(8 * L, dtype=np.int32)
        _check(lib().ref_derive_patch_spec(C.c_void_p(self.h), _p(r), _p(out)))
        return out[:4 * L].reshape(L, 4), out[4 * L:].reshape(L, 4)


class PatchRunner:
    """Reference PatchRunner (proj/src/runtime.cpp:110-476)."""

    ENTRIES = {"run_step": 0, "reference": 1, "naive": 2, "sync": 3, "displaced": 4}

    def __init__(self, model, cond, h, w, mode="reference", n_devices=1, warmup=4,
                 gn_scheme="corrected", stress=False):
        cond = f32(cond)
        self.model = model
        self.h, self.w = h, w
        r = lib().ref_runner_create(C.c_void_p(model.h), _p(cond), len(cond), h, w,
                                    MODES[mode], n_devices, warmup, GN_SCHEMES[gn_scheme],
                                    int(stress))
        if not r:
            raise RefInvalidArgument(1, lib().ref_last_error().decode())
        self.r = r

    def __del__(self):
        if getattr(self, "r", None) and _lib is not None:
            _lib.ref_runner_free(self.r)

    def step(self, entry, x, t, step_index):
        x = f32(x)
        eps = np.zeros_like(x)
        _check(lib().ref_runner_step(C.c_void_p(self.r), self.ENTRIES[entry], _p(x), x.shape[1],
                                     x.shape[2], x.shape[3], t, step_index, _p(eps)))
        return eps

    def cached_input(self, dev, layer):
        s = np.zeros(4, dtype=np.int32)
        n = lib().ref_runner_cached_input(C.c_void_p(self.r), dev, layer, None, _p(s))
        if n == 0:
            return None
        a = np.zeros(tuple(int(v) for v in s), dtype=np.float32)
        lib().ref_runner_cached_input(C.c_void_p(self.r), dev, layer, _p(a), _p(s))
        return a

    def total_macs(self):
        return int(lib().ref_runner_total_macs(C.c_void_p(self.r)))

    def volumes(self):
        v = np.zeros(6, dtype=np.uint64)
        lib().ref_runner_volumes(C.c_void_p(self.r), _p(v))
        return [int(x) for x in v]

    def trace(self, dev=0):
        """PatchRunner::trace() (runtime.hpp:71) rows: (device, step, layer, kind, prim, macs,
        bytes_recv, bytes_sent, tag)."""
        f = lib().ref_runner_trace
        f.restype = C.c_long
        f.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_long]
        n = f(C.c_void_p(self.r), dev, None, 0)
        out = np.zeros((max(n, 1), 9), dtype=np.uint64)
        f(C.c_void_p(self.r), dev, _p(out), n)
        rows = []
        for r in out[:n]:
            v = [int(x) for x in r]
            v[2] = v[2] - (1 << 64) if v[2] >= (1 << 63) else v[2]
            rows.append(tuple(v))
        return rows


def run_sampling(cfg6, mode="reference", n_devices=1, h=48, w=48, num_steps=50, warmup=4,
                 gn_scheme="corrected", stress=False, seeds=(42, 1234, 7),
                 schedule_steps=1000, beta_start=1e-4, beta_end=2e-2, trajectory=False):
    """Reference run_sampling (proj/src/runtime.cpp:494-526)."""
    c6 = np.array(cfg6, dtype=np.int32)
    ic = np.array([MODES[mode], n_devices, h, w, num_steps, warmup, GN_SCHEMES[gn_scheme],
                   int(stress), schedule_steps], dtype=np.int32)
    sd = np.array(seeds, dtype=np.uint64)
    x0 = np.zeros((1, cfg6[0], h, w), dtype=np.float32)
    traj = np.zeros((num_steps, 1, cfg6[0], h, w), dtype=np.float32) if trajectory else None
    macs = np.zeros(1, dtype=np.uint64)
    vol = np.zeros(6, dtype=np.uint64)
    _check(lib().ref_run_sampling(_p(c6), _p(ic), _p(sd), beta_start, beta_end, _p(x0),
                                  _p(traj) if traj is not None else None, _p(macs), _p(vol)))
    return {"x0": x0, "trajectory": traj, "total_macs": int(macs[0]),
            "volumes": [int(v) for v in vol]}


# ---- kernel-level wrappers (proj/src/tensor.cpp) --------------------------------------
def conv2d_region(x, region, weight, bias, stride, pad):
    x, weight, bias = f32(x), f32(weight), f32(bias)
    n, c, h, w = x.shape
    r0, r1 = region[0], region[1]
    k = weight.shape[2]
    out_h = (h + 2 * pad - k) // stride + 1
    out_w = (w + 2 * pad - k) // stride + 1
    oy0 = min(-(-r0 // stride), out_h)
    oy1 = min(-(-r1 // stride), out_h)
    out = np.zeros((n, weight.shape[0], max(oy1 - oy0, 0), out_w), dtype=np.float32)
    _check(lib().ref_conv2d_region(_p(x), n, c, h, w, r0, r1, _p(weight), weight.shape[0], k,
                                   _p(bias), stride, pad, _p(out)))
    return out


def attention(q, k, v, scale):
    q, k, v = f32(q), f32(k), f32(v)
    n, _, m, d = q.shape
    s, dv = k.shape[2], v.shape[3]
    out = np.zeros((n, 1, m, dv), dtype=np.float32)
    _check(lib().ref_attention(_p(q), _p(k), _p(v), n, m, s, d, dv, scale, _p(out)))
    return out


def linear(tokens, weight, bias):
    tokens, weight, bias = f32(tokens), f32(weight), f32(bias)
    n, _, t, i = tokens.shape
    o = weight.shape[0]
    out = np.zeros((n, 1, t, o), dtype=np.float32)
    _check(lib().ref_linear(_p(tokens), n, t, i, _p(weight), o, _p(bias), _p(out)))
    return out


def group_stats(x, groups, region=None):
    x = f32(x)
    n, c, h, w = x.shape
    mean = np.zeros(n * groups)
    msq = np.zeros(n * groups)
    r0, r1 = (region[0], region[1]) if region is not None else (-1, -1)
    _check(lib().ref_group_stats(_p(x), n, c, h, w, groups, r0, r1, _p(mean), _p(msq)))
    return mean, msq


def group_norm_apply(x, region, mean, mean_sq, gamma, beta, eps):
    x, gamma, beta = f32(x), f32(gamma), f32(beta)
    n, c, h, w = x.shape
    mean = np.ascontiguousarray(mean, dtype=np.float64)
    mean_sq = np.ascontiguousarray(mean_sq, dtype=np.float64)
    out = np.zeros_like(x)
    r0, r1 = (region[0], region[1]) if region is not None else (-1, -1)
    _check(lib().ref_group_norm_apply(_p(x), n, c, h, w, r0, r1, len(mean) // n, _p(mean),
                                      _p(mean_sq), _p(gamma), _p(beta), eps, _p(out)))
    return out


def corrected_gn_stats(fresh, prev_local, prev_global):
    g = len(fresh[0])
    arr = [np.ascontiguousarray(np.concatenate(s), dtype=np.float64)
           for s in (fresh, prev_local, prev_global)]
    out = np.zeros(2 * g)
    _check(lib().ref_corrected_gn_stats(g, _p(arr[0]), _p(arr[1]), _p(arr[2]), _p(out)))
    return out[:g], out[g:]


def silu(x):
    x = f32(x)
    out = np.zeros_like(x)
    _check(lib().ref_silu(_p(x), x.size, _p(out)))
    return out


def upsample_nearest2x(x):
    x = f32(x)
    n, c, h, w = x.shape
    out = np.zeros((n, c, 2 * h, 2 * w), dtype=np.float32)
    _check(lib().ref_upsample(_p(x), n, c, h, w, _p(out)))
    return out


def random_normal(n, c, h, w, seed):
    out = np.zeros((n, c, h, w), dtype=np.float32)
    _check(lib().ref_random_normal(n, c, h, w, seed, _p(out)))
    return out


def random_condition(dim, seed):
    out = np.zeros(dim, dtype=np.float32)
    _check(lib().ref_random_condition(dim, seed, _p(out)))
    return out


def timestep_embedding(t, dim):
    out = np.zeros(dim, dtype=np.float32)
    _check(lib().ref_timestep_embedding(t, dim, _p(out)))
    return out


def make_schedule(total=1000, b0=1e-4, b1=2e-2):
    out = np.zeros(total)
    _check(lib().ref_make_schedule(total, b0, b1, _p(out)))
    return out


def make_plan(total, steps):
    out = np.zeros(steps, dtype=np.int32)
    _check(lib().ref_make_plan(total, steps, _p(out)))
    return [int(v) for v in out]


def ddim_update(x, eps, abar_t, abar_n):
    x, eps = f32(x), f32(eps)
    out = np.zeros_like(x)
    _check(lib().ref_ddim_update(_p(x), _p(eps), x.size, abar_t, abar_n, _p(out)))
    return out


def partition_rows(h, n, w):
    out = np.zeros(4 * n, dtype=np.int32)
    _check(lib().ref_partition_rows(h, n, w, _p(out)))
    return [tuple(int(v) for v in out[4 * i:4 * i + 4]) for i in range(n)]


def run_config_validate(cfg6, mode, n_devices, h, w, num_steps=50, warmup=4):
    c6 = np.array(cfg6, dtype=np.int32)
    ic = np.array([MODES[mode], n_devices, h, w, num_steps, warmup, 0, 0, 1000], dtype=np.int32)
    _check(lib().ref_run_config_validate(_p(c6), _p(ic)))


def fnv1a64(arr):
    """FNV-1a over the float bytes, proj/tests/test_model.cpp:26-37."""
    h = 1469598103934665603
    for b in np.ascontiguousarray(arr, dtype=np.float32).tobytes():
        h ^= b
        h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return h

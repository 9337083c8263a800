"""ctypes binding of ``libpp_b200.so`` (the C ABI declared in ``include/pp_b200.h``).

The library is built in-tree (``paper_2402_19481_b200/build.py``).  There is no
Python or CPU fallback: if the library cannot be loaded, or no B200 is present,
calls fail loudly.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PP_B200_LIB") or os.path.join(HERE, "libpp_b200.so")

PP_OK, PP_EINVAL, PP_ERUNTIME, PP_ECUDA, PP_ENCCL = 0, 1, 2, 3, 4
DTYPES = {"bf16": 0, "fp32": 1}
MODES = {"reference": 0, "naive": 1, "sync-pp": 2, "displaced": 3}
GN_SCHEMES = {"corrected": 0, "stale": 1, "separate": 2}
TRANSPORTS = {"nccl": 0, "ipc": 1}
ENTRIES = {"run_step": 0, "reference": 1, "naive": 2, "sync": 3, "displaced": 4}


class PPError(Exception):
    code = None


class InvalidArgument(PPError, ValueError):
    """std::invalid_argument in the reference (CLI exit 2)."""
    code = PP_EINVAL


class RuntimeFailure(PPError, RuntimeError):
    """std::runtime_error in the reference (CLI exit 1)."""
    code = PP_ERUNTIME


class CudaError(PPError, RuntimeError):
    code = PP_ECUDA


class NcclError(PPError, RuntimeError):
    code = PP_ENCCL


_ERRS = {PP_EINVAL: InvalidArgument, PP_ERUNTIME: RuntimeFailure, PP_ECUDA: CudaError,
         PP_ENCCL: NcclError}

_lib = None
_lock = threading.Lock()


class ModelConfig(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("in_channels", "base_channels", "levels", "groups",
                                        "cond_dim", "attn_at_level", "res_blocks", "attn_levels",
                                        "attn_depth", "attn_up")]


class LayerDesc(C.Structure):
    _fields_ = [("id", C.c_int), ("kind", C.c_int), ("in_ch", C.c_int), ("out_ch", C.c_int),
                ("kernel", C.c_int), ("stride", C.c_int), ("pad", C.c_int), ("groups", C.c_int),
                ("eps", C.c_float), ("cond_dim", C.c_int), ("skip_source", C.c_int),
                ("scale_in", C.c_int), ("scale_out", C.c_int), ("weight", C.c_int),
                ("bias", C.c_int), ("weight2", C.c_int), ("bias2", C.c_int)]


class RunConfig(C.Structure):
    _fields_ = [("mode", C.c_int), ("n_devices", C.c_int), ("h", C.c_int), ("w", C.c_int),
                ("num_steps", C.c_int), ("warmup", C.c_int), ("gn_scheme", C.c_int),
                ("dtype", C.c_int), ("model_seed", C.c_uint64), ("noise_seed", C.c_uint64),
                ("cond_seed", C.c_uint64), ("model", ModelConfig), ("schedule_steps", C.c_int),
                ("beta_start", C.c_double), ("beta_end", C.c_double)]


class RunnerOpts(C.Structure):
    _fields_ = [("mode", C.c_int), ("n_devices", C.c_int), ("warmup_steps", C.c_int),
                ("gn_scheme", C.c_int), ("dtype", C.c_int), ("world", C.c_int),
                ("rank", C.c_int), ("nccl_id", C.c_void_p), ("device", C.c_int),
                ("profile", C.c_int), ("transport", C.c_int), ("no_comm", C.c_int),
                ("stress", C.c_int), ("stress_seed", C.c_ulonglong),
                ("cfg_scale", C.c_double), ("uncond", C.c_void_p), ("cfg_nccl_id", C.c_void_p),
                ("cond_tokens", C.c_int), ("cfg_pair_role", C.c_int), ("cfg_pair_transport", C.c_int)]


_V, _I, _L, _D, _U64, _F = C.c_void_p, C.c_int, C.c_long, C.c_double, C.c_uint64, C.c_float
_LL, _SZ = C.c_longlong, C.c_size_t

# name: (restype, argtypes)
SIGNATURES = {
    "pp_last_error": (C.c_char_p, []),
    "pp_version": (_I, []),
    "pp_set_pdl": (None, [_I]),
    "pp_device_count": (_I, []),
    "pp_model_build": (_I, [_V, _U64, _V]),
    "pp_model_from_pool": (_I, [_V, _V, _SZ, _V]),
    "pp_model_destroy": (None, [_V]),
    "pp_model_num_layers": (_I, [_V]),
    "pp_model_layer": (_I, [_V, _I, _V]),
    "pp_model_num_weights": (_I, [_V]),
    "pp_model_weight_shape": (_I, [_V, _I, _V]),
    "pp_model_pool_size": (_SZ, [_V]),
    "pp_model_pool": (_I, [_V, _V]),
    "pp_model_zero_weights": (_I, [_V, _I]),
    "pp_model_total_macs": (_U64, [_V, _I, _I]),
    "pp_partition_rows": (_I, [_I, _I, _I, _V]),
    "pp_derive_patch_spec": (_I, [_V, _V, _V, _V]),
    "pp_corrected_gn_stats": (_I, [_I, _V, _V, _V, _V]),
    "pp_run_config_default": (None, [_V]),
    "pp_run_config_validate": (_I, [_V]),
    "pp_make_schedule": (_I, [_I, _D, _D, _V]),
    "pp_make_plan": (_I, [_I, _I, _V]),
    "pp_random_normal": (_I, [_I, _I, _I, _I, _U64, _V]),
    "pp_random_condition": (_I, [_I, _U64, _V]),
    "pp_macs_of_layer": (_U64, [_V, _I, _V]),
    "pp_runner_opts_default": (None, [_V]),
    "pp_runner_create": (_I, [_V, _V, _I, _I, _I, _V, _V]),
    "pp_runner_destroy": (None, [_V]),
    "pp_runner_step": (_I, [_V, _I, _V, _I, _I, _V]),
    "pp_runner_patch_spec": (_I, [_V, _I, _V, _V]),
    "pp_runner_cached_input": (_L, [_V, _I, _I, _V, _V]),
    "pp_runner_total_macs": (_U64, [_V]),
    "pp_runner_step_device_macs": (_I, [_V, _I, _V]),
    "pp_runner_volumes": (_I, [_V, _V]),
    "pp_runner_trace": (_L, [_V, _I, _V, _L]),
    "pp_runner_sample": (_I, [_V, _V, _V, _I, _V, _I, _V, _V]),
    "pp_runner_profile": (_I, [_V, _V]),
    "pp_runner_launches": (_L, [_V]),
    "pp_runner_last_device_ms": (_D, [_V]),
    "pp_runner_set_profile": (_I, [_V, _I]),
    "pp_nccl_unique_id": (_I, [_V]),
    "pp_runner_ipc_export": (_I, [_V, _V, _L, _V]),
    "pp_runner_ipc_connect": (_I, [_V, _V, _L]),
    "pp_runner_pair_export": (_I, [_V, _V, _L, _V]),
    "pp_runner_pair_connect": (_I, [_V, _V, _L]),
    "pp_assemble_bands": (_I, [_V, _I, _I, _I, _I, _V]),
    "pp_dev_gemm_bench": (_I, [_I, _I, _I, _I, _I, _I, _I, _I, _I, _V]),
    "pp_dev_gn_bench": (_I, [_I, _LL, _I, _I, _I, _I, _V]),
    "pp_run_sampling": (_I, [_V, _V, _V, _V]),
    "pp_conv2d_region": (_I, [_I, _V, _I, _I, _I, _I, _I, _I, _V, _I, _I, _V, _I, _I, _V]),
    "pp_linear": (_I, [_I, _V, _I, _I, _I, _V, _I, _V, _V]),
    "pp_attention": (_I, [_I, _V, _V, _V, _I, _I, _I, _I, _I, _F, _V]),
    "pp_group_stats": (_I, [_I, _V, _I, _I, _I, _I, _I, _I, _I, _V, _V]),
    "pp_group_norm_apply": (_I, [_I, _V, _I, _I, _I, _I, _I, _I, _I, _V, _V, _V, _V, _F, _V]),
    "pp_silu": (_I, [_I, _V, _L, _V]),
    "pp_upsample_nearest2x": (_I, [_I, _V, _I, _I, _I, _I, _V]),
    "pp_ddim_update": (_I, [_V, _V, _L, _D, _D, _V]),
    "pp_dev_gemm": (_I, [_I, _V, _I, _I, _LL, _V, _I, _LL, _V, _V, _LL, _I, _I, _I, _V]),
    "pp_dev_conv": (_I, [_I, _V, _I, _I, _I, _I, _V, _I, _I, _V, _V, _LL, _I, _V, _LL, _I, _I,
                         _V]),
}


def build_if_needed():
    if os.path.exists(LIB_PATH):
        return
    from . import build as _b
    _b.build()


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build_if_needed()
            L = C.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                f = getattr(L, name, None)
                if f is None:      # reported by tests/test_abi.py
                    continue
                f.restype = res
                f.argtypes = args
            _lib = L
    return _lib


def last_error():
    return lib().pp_last_error().decode()


def check(rc):
    if rc != PP_OK:
        raise _ERRS.get(rc, PPError)(last_error())
    return rc

"""ctypes binding of the in-tree C-ABI library ``libdasmc_gpu.so``.

The product path has no CPU fallback: if the shared library (built by
``__graft_entry__.build()`` / ``make -C paper_2601_21983_b200``) is missing,
importing the high-level API raises.  Declarations mirror
``include/dasmc_gpu.h`` one to one.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# DASMC_GPU_LIB overrides the library path (profiling builds of the same sources)
LIB_PATH = os.environ.get("DASMC_GPU_LIB") or os.path.join(_HERE, "libdasmc_gpu.so")

DASMC_OK, DASMC_EINVAL, DASMC_EDEAD, DASMC_ECUDA = 0, -1, -2, -3
RELU, TANH = 0, 1
SCALED, SDA = 0, 1
HMC, LANGEVIN = 0, 1
MULTINOMIAL, SYSTEMATIC = 0, 1
PREC_FP32, PREC_TF32, PREC_3XTF32, PREC_F16, PREC_TF32H, PREC_F16X2 = 0, 1, 2, 3, 4, 5
SCHED_CONSTANT, SCHED_FULL_BATCH, SCHED_CTR, SCHED_LINEAR, SCHED_AUTOMATED, SCHED_SDA = range(6)


class NetDesc(C.Structure):
    _fields_ = [("num_layers", C.c_int), ("layer_sizes", C.POINTER(C.c_int)), ("activation", C.c_int),
                ("conv", C.POINTER(C.c_int))]


class KernelCfg(C.Structure):
    _fields_ = [("step_size", C.c_double), ("leapfrog_steps", C.c_int), ("kind", C.c_int)]


class IterRecord(C.Structure):
    _fields_ = [
        ("k", C.c_int),
        ("batch", C.c_int64),
        ("beta", C.c_double),
        ("ess", C.c_double),
        ("resampled", C.c_int),
        ("mean_log_target", C.c_double),
        ("sampler_ms", C.c_double),
        ("n_divergent", C.c_int),
    ]


class Schedule(C.Structure):
    _fields_ = [
        ("kind", C.c_int),
        ("initial_batch", C.c_int64),
        ("increment", C.c_int64),
        ("iterations", C.c_int),
        ("dataset_size", C.c_int64),
        ("period", C.c_int),
        ("switch_iteration", C.c_int),
    ]


class SdaState(C.Structure):
    _fields_ = [
        ("beta", C.c_double),
        ("entropy_step", C.c_double),
        ("beta_reset", C.c_double),
        ("prefix_end", C.c_int64),
        ("block_end", C.c_int64),
        ("total_n", C.c_int64),
        ("stage", C.c_int),
        ("terminal", C.c_int),
    ]


class RunCfg(C.Structure):
    _fields_ = [
        ("kernel", KernelCfg),
        ("schedule", Schedule),
        ("sigma", C.c_double),
        ("beta0", C.c_double),
        ("entropy_step", C.c_double),
        ("particles", C.c_int),
        ("iterations", C.c_int),
        ("seed", C.c_uint64),
        ("resample_fraction", C.c_double),
        ("resample_kind", C.c_int),
        ("resample_always", C.c_int),
        ("redraw_constant", C.c_int),
    ]


_P = C.c_void_p
_D = C.POINTER(C.c_double)
_F = C.POINTER(C.c_float)
_I32 = C.POINTER(C.c_int32)
_I64 = C.POINTER(C.c_int64)

# name -> (restype, argtypes)
SIGNATURES = {
    "dasmc_last_error": (C.c_char_p, []),
    "dasmc_gpu_create": (C.c_int, [C.POINTER(NetDesc), _F, _I32, C.c_int64, C.c_int, C.c_int, C.c_int, C.POINTER(_P)]),
    "dasmc_gpu_destroy": (C.c_int, [_P]),
    "dasmc_gpu_param_count": (C.c_int, [_P]),
    "dasmc_gpu_set_target": (C.c_int, [_P, C.c_int64, C.c_int64, C.c_int64, C.c_int, C.c_double, C.c_double]),
    "dasmc_gpu_value_and_grad": (C.c_int, [_P, _D, C.c_int64, _D, _D]),
    "dasmc_gpu_loglik_parts": (C.c_int, [_P, _D, C.c_int64, _D, _D]),
    "dasmc_gpu_momentum": (C.c_int, [_P, C.c_uint64, C.c_int, C.c_int64, _D]),
    "dasmc_gpu_resample_indices": (C.c_int, [_P, _D, _D, C.c_int64, C.c_int, _I32]),
    "dasmc_gpu_uniforms": (C.c_int, [_P, C.c_uint64, C.c_int, C.c_int64, _D]),
    "dasmc_gpu_create_multi": (C.c_int, [C.POINTER(NetDesc), _F, _I32, C.c_int64, C.c_int, C.POINTER(C.c_int), C.c_int,
                                          C.c_int, C.POINTER(_P)]),
    "dasmc_gpu_multi_shards": (C.c_int, [_P]),
    "dasmc_gpu_set_graphs": (C.c_int, [_P, C.c_int]),
    "dasmc_gpu_init_ensemble": (C.c_int, [_P, C.c_int64, C.c_uint64]),
    "dasmc_gpu_set_ensemble": (C.c_int, [_P, _D, _D, C.c_int64, C.c_int]),
    "dasmc_gpu_get_ensemble": (C.c_int, [_P, _D, _D, C.POINTER(C.c_int)]),
    "dasmc_gpu_set_ensemble_f32": (C.c_int, [_P, _F, _D, C.c_int64, C.c_int]),
    "dasmc_gpu_get_ensemble_f32": (C.c_int, [_P, _F, _D, C.POINTER(C.c_int)]),
    "dasmc_gpu_smc_step": (C.c_int, [_P, C.POINTER(KernelCfg), C.c_uint64, C.c_int, C.c_double, C.c_int, C.POINTER(IterRecord)]),
    "dasmc_gpu_sync_records": (C.c_int, [_P, C.POINTER(IterRecord), C.c_int]),
    "dasmc_gpu_last_proposals": (C.c_int, [_P, _D, _D, _D, _I32, _D, _I32]),
    "dasmc_gpu_sda_moments": (C.c_int, [_P, C.c_int64, C.c_int64, _D]),
    "dasmc_batch_size": (C.c_int64, [C.POINTER(Schedule), C.c_int]),
    "dasmc_sda_init": (C.c_int, [C.POINTER(Schedule), C.c_double, C.c_double, C.POINTER(SdaState)]),
    "dasmc_sda_beta_step": (C.c_double, [C.c_double, _D, C.c_double]),
    "dasmc_sda_advance_with": (C.c_int, [C.POINTER(Schedule), C.POINTER(SdaState), _D]),
    "dasmc_sda_moments_from": (C.c_int, [_D, _D, _D, C.c_int64, _D]),
    "dasmc_make_teacher_data": (C.c_int, [C.POINTER(NetDesc), C.c_int64, C.c_int, C.c_uint64, C.c_uint64, C.c_int, _F, _I32]),
    "dasmc_shuffle_permutation": (C.c_int, [C.c_uint64, C.c_int64, _I64]),
    "dasmc_shard_range": (None, [C.c_int64, C.c_int, C.c_int, _I64, _I64]),
    "dasmc_gpu_init_ensemble_at": (C.c_int, [_P, C.c_int64, C.c_uint64, C.c_int64]),
    "dasmc_shard_plan": (C.c_int, [_I32, C.c_int64, C.c_int, C.c_int, _I32, _I32, _I64, _I32]),
    "dasmc_gpu_shard_propose": (C.c_int, [_P, C.POINTER(KernelCfg), C.c_uint64, C.c_int64, C.c_void_p, C.c_void_p]),
    "dasmc_gpu_shard_resample": (C.c_int, [_P, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_uint64, C.c_int,
                                           C.c_double, C.c_int, C.c_void_p, C.POINTER(IterRecord)]),
    "dasmc_gpu_row_floats": (C.c_int64, [_P]),
    "dasmc_gpu_pack_rows": (C.c_int, [_P, _I32, C.c_int64, C.c_void_p]),
    "dasmc_gpu_unpack_rows": (C.c_int, [_P, C.c_void_p, _I32, C.c_int64]),
    "dasmc_gpu_reserve_rows": (C.c_int, [_P, C.c_int64]),
    "dasmc_gpu_stream": (C.c_void_p, [_P]),
    "dasmc_launch_count": (C.c_int64, []),
    "dasmc_gpu_set_timing": (C.c_int, [_P, C.c_int]),
    "dasmc_gpu_kernel_times": (C.c_int, [_P, _D, _I64]),
    "dasmc_gpu_bench_memory": (C.c_int, [_P, C.c_int64, _I32, C.c_int, _D, _D]),
    "dasmc_rng_skip": (C.c_int, [C.c_uint64, C.c_uint64, C.c_int64, C.POINTER(C.c_uint64)]),
    "dasmc_gpu_evaluate_predictive": (C.c_int, [_P, _F, _I32, C.c_int64, _D, _D]),
    "dasmc_gpu_predictive_mix": (C.c_int, [_P, _F, _I32, C.c_int64, _D, C.c_int64, _D]),
    "dasmc_predictive_metrics": (C.c_int, [_D, _I32, C.c_int64, C.c_int, _D, _D]),
    "dasmc_parse_idx": (C.c_int, [C.c_char_p, C.c_int64, C.c_char_p, C.c_int64, _I64, _I64, C.POINTER(C.c_int), _F,
                                  _I32]),
    "dasmc_load_idx": (C.c_int, [C.c_char_p, C.c_char_p, _I64, _I64, C.POINTER(C.c_int), _F, _I32]),
    "dasmc_make_synthetic": (C.c_int, [C.c_int, C.c_int64, C.c_double, C.c_uint64, _F, _I32]),
    "dasmc_redraw_rows": (C.c_int, [C.c_uint64, C.c_int, C.c_int64, C.c_int64, _I64]),
    "dasmc_gpu_set_rows": (C.c_int, [_P, _I64, C.c_int64]),
    "dasmc_gpu_set_cache_start": (C.c_int, [_P, C.c_int]),
    "dasmc_gpu_last_step_cached": (C.c_int, [_P]),
    "dasmc_gpu_run": (C.c_int, [C.POINTER(NetDesc), _F, _I32, C.c_int64, C.POINTER(RunCfg), C.c_int, C.c_int,
                                C.POINTER(IterRecord), C.POINTER(SdaState), _D, _D]),
}

_lib = None


_alt = {}


def load(path: str = LIB_PATH) -> C.CDLL:
    """Load the product library (raises if it has not been built).  A path other than
    LIB_PATH loads a second build of the same sources side by side (A/B timing tools)."""
    global _lib
    if path != LIB_PATH:
        if path not in _alt:
            _alt[path] = _bind(path)
        return _alt[path]
    if _lib is not None:
        return _lib
    _lib = _bind(path)
    return _lib


def _bind(path: str) -> C.CDLL:
    if not os.path.exists(path):
        raise RuntimeError(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback for the product path)")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


class DasmcError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class SamplerError(DasmcError):
    """All particles dead (smc.hpp:21-24)."""


def check(rc: int) -> None:
    if rc == DASMC_OK:
        return
    # the message of whichever loaded build failed (A/B tools load a second build)
    msgs = [lib.dasmc_last_error().decode() for lib in [load(), *_alt.values()]]
    msg = next((m for m in msgs if m), "")
    if rc == DASMC_EDEAD:
        raise SamplerError(rc, msg)
    if rc == DASMC_EINVAL:
        raise ValueError(msg)
    raise DasmcError(rc, msg)

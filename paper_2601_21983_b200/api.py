"""Python mirror of the reference's sampler / schedule API over the C-ABI.

Names follow the reference (``/root/reference/proj/include/dasmc``):
``NetSpec``, ``KernelConfig``, ``ScheduleConfig``, ``log_target_with_grad``,
``init_ensemble``, ``smc_step``, ``batch_size``, ``sda_advance`` ...  The only
structural difference is the seam: calls act on the whole particle ensemble
(see include/dasmc_gpu.h), so per-particle inputs are ``[J, D]`` arrays in the
reference parameter layout.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _lib as L

_PREC = {"fp32": L.PREC_FP32, "tf32": L.PREC_TF32, "3xtf32": L.PREC_3XTF32, "f16": L.PREC_F16, "tf32h": L.PREC_TF32H, "f16x2": L.PREC_F16X2}
_SCHED = {"constant": L.SCHED_CONSTANT, "full_batch": L.SCHED_FULL_BATCH, "ctr": L.SCHED_CTR,
          "linear": L.SCHED_LINEAR, "automated": L.SCHED_AUTOMATED, "sda": L.SCHED_SDA}
_RESAMPLE = {"multinomial": L.MULTINOMIAL, "systematic": L.SYSTEMATIC}


def _dp(a):
    return a.ctypes.data_as(L._D) if a is not None else None


def _fp(a):
    return a.ctypes.data_as(L._F) if a is not None else None


def _ip(a):
    return a.ctypes.data_as(L._I32) if a is not None else None


@dataclass
class NetSpec:  # network.hpp:24-27
    """layer_sizes: the MLP {input, hidden..., classes}.  [EXT] conv: a CNN front
    ((c, h, w), [(k, cout, pool), ...]) whose flattened output feeds the MLP, so
    layer_sizes[0] must be the flatten size (include/dasmc_gpu.h)."""
    layer_sizes: Sequence[int]
    activation: str = "relu"
    conv: Optional[tuple] = None

    def conv_array(self):
        if self.conv is None:
            return None
        (c, h, w), stages = self.conv
        v = [c, h, w, len(stages)]
        for k, co, pool in stages:
            v += [k, co, 1 if pool else 0]
        return v

    def input_dim(self) -> int:
        if self.conv is None:
            return int(self.layer_sizes[0])
        c, h, w = self.conv[0]
        return c * h * w

    def desc(self):
        arr = (C.c_int * len(self.layer_sizes))(*self.layer_sizes)
        cv = self.conv_array()
        carr = (C.c_int * len(cv))(*cv) if cv is not None else None
        d = L.NetDesc(len(self.layer_sizes), arr, L.RELU if self.activation == "relu" else L.TANH, carr)
        d._keep = (arr, carr)
        return d

    def oracle_layers(self):
        """The oracle's model encoding (oracle/pyoracle.py cnn_layers) -- tests only."""
        if self.conv is None:
            return list(self.layer_sizes)
        (c, h, w), stages = self.conv
        out = [-1, c, h, w, len(stages)]
        for k, co, pool in stages:
            out += [k, co, 1 if pool else 0]
        return out + list(self.layer_sizes)


def conv_param_count(spec: NetSpec) -> int:
    if spec.conv is None:
        return 0
    (c, h, w), stages = spec.conv
    total = 0
    for k, co, pool in stages:
        total += co * c * k * k + co
        h, w = h - k + 1, w - k + 1
        if pool:
            h, w = h // 2, w // 2
        c = co
    return total


def param_count(spec: NetSpec) -> int:  # network.hpp:36-42 (+ [EXT] conv blocks)
    s = list(spec.layer_sizes)
    if len(s) < 2 or min(s) < 1:
        raise ValueError("NetSpec: invalid layer sizes")
    return conv_param_count(spec) + sum(s[i - 1] * s[i] + s[i] for i in range(1, len(s)))


@dataclass
class KernelConfig:  # kernels.hpp:26-49
    step_size: float
    leapfrog_steps: int = 1
    kind: str = "hmc"

    @staticmethod
    def hmc(h, s):
        return KernelConfig(h, s, "hmc")

    @staticmethod
    def langevin(h):
        return KernelConfig(h, 1, "langevin")

    def c(self):
        return L.KernelCfg(self.step_size, self.leapfrog_steps, L.HMC if self.kind == "hmc" else L.LANGEVIN)


@dataclass
class ScheduleConfig:  # annealing.hpp:23-30 (+ [EXT] period, switch_iteration)
    kind: str = "full_batch"
    initial_batch: int = 1
    increment: int = 1
    iterations: int = 1
    dataset_size: int = 1
    period: int = 1
    switch_iteration: int = -1

    def c(self):
        return L.Schedule(_SCHED[self.kind], self.initial_batch, self.increment, self.iterations,
                          self.dataset_size, self.period, self.switch_iteration)


def batch_size(cfg: ScheduleConfig, k: int) -> int:  # annealing.hpp:52-82
    lib = L.load()
    s = cfg.c()
    v = lib.dasmc_batch_size(C.byref(s), k)
    if v < 0:
        raise ValueError(lib.dasmc_last_error().decode())
    return int(v)


def sda_beta_step(beta: float, entropy_step: float, denom: float):  # annealing.hpp:114-122
    st = C.c_double(entropy_step)
    b = L.load().dasmc_sda_beta_step(beta, C.byref(st), denom)
    return b, st.value


def sda_init(cfg: ScheduleConfig, beta0=0.1, entropy_step=1.0) -> L.SdaState:
    out = L.SdaState()
    s = cfg.c()
    L.check(L.load().dasmc_sda_init(C.byref(s), beta0, entropy_step, C.byref(out)))
    return out


def sda_advance_with(cfg: ScheduleConfig, state: L.SdaState, moments6) -> L.SdaState:
    st = L.SdaState.from_buffer_copy(state)
    m = np.ascontiguousarray(moments6, dtype=np.float64)
    s = cfg.c()
    L.check(L.load().dasmc_sda_advance_with(C.byref(s), C.byref(st), _dp(m)))
    return st


def sda_moments_from(prefix_nll, block_nll, log_weights) -> np.ndarray:
    a, b, w = (np.ascontiguousarray(x, dtype=np.float64) for x in (prefix_nll, block_nll, log_weights))
    out = np.zeros(6)
    L.check(L.load().dasmc_sda_moments_from(_dp(a), _dp(b), _dp(w), len(a), _dp(out)))
    return out


def make_teacher_data(spec: NetSpec, n: int, feature_kind: int, seed: int, cfg_id: int, threads: int = 8):
    """[EXT] teacher-labelled synthetic data; X fp32 [n, d], y int32 [n]."""
    X = np.empty((n, spec.input_dim()), dtype=np.float32)
    y = np.empty(n, dtype=np.int32)
    d = spec.desc()
    L.check(L.load().dasmc_make_teacher_data(C.byref(d), n, feature_kind, seed, cfg_id, threads, _fp(X), _ip(y)))
    return X, y


def _idx(call):
    n, d, nc = C.c_int64(), C.c_int64(), C.c_int()
    L.check(call(C.byref(n), C.byref(d), C.byref(nc), None, None))
    X = np.empty((n.value, d.value), dtype=np.float32)
    y = np.empty(n.value, dtype=np.int32)
    L.check(call(C.byref(n), C.byref(d), C.byref(nc), _fp(X), _ip(y)))
    return X, y, nc.value


def parse_idx(image_bytes: bytes, label_bytes: bytes):  # dataset.hpp:84-131
    """(X [n, rows*cols] fp32 pixels/255, y int32, num_classes) from IDX byte streams."""
    return _idx(lambda n, d, nc, X, y: L.load().dasmc_parse_idx(image_bytes, len(image_bytes), label_bytes,
                                                                len(label_bytes), n, d, nc, X, y))


def load_idx(image_path: str, label_path: str):  # dataset.hpp:186-196 (gzip transparent)
    return _idx(lambda n, d, nc, X, y: L.load().dasmc_load_idx(image_path.encode(), label_path.encode(), n, d, nc,
                                                               X, y))


def redraw_rows(seed: int, k: int, n: int, count: int) -> np.ndarray:  # runner.hpp:531-542
    r = np.empty(count, dtype=np.int64)
    L.check(L.load().dasmc_redraw_rows(seed, k, n, count, r.ctypes.data_as(L._I64)))
    return r


def shuffle_permutation(seed: int, n: int) -> np.ndarray:  # runner.hpp:486-489
    p = np.empty(n, dtype=np.int64)
    L.check(L.load().dasmc_shuffle_permutation(seed, n, p.ctypes.data_as(L._I64)))
    return p


def _rec(r: L.IterRecord) -> dict:
    return {"k": r.k, "batch": r.batch, "beta": r.beta, "ess": r.ess, "resampled": bool(r.resampled),
            "mean_log_target": r.mean_log_target, "sampler_ms": r.sampler_ms, "n_divergent": r.n_divergent}


class GpuEnsembleTarget:
    """Device-resident dataset + TargetContext + ParticleEnsemble on one B200.

    Replaces the reference's per-particle ``ContextTarget`` (target.hpp:180-190)
    and the ensemble loop of ``smc_step`` (smc.hpp:109-158)."""

    def __init__(self, spec: NetSpec, X: np.ndarray, y: np.ndarray, max_particles: int, device: int = 0,
                 precision: str = "fp32", lib_path: str | None = None, devices: Optional[Sequence[int]] = None):
        """devices: a single-process multi-GPU group (dasmc_gpu_create_multi): the ensemble is
        sharded over one shard context per listed device (devices may repeat)."""
        self.lib = L.load(lib_path) if lib_path else L.load()
        self.spec = spec
        self.D = param_count(spec)
        X = np.ascontiguousarray(X, dtype=np.float32)
        y = np.ascontiguousarray(y, dtype=np.int32)
        self.n = X.shape[0]
        d = spec.desc()
        h = C.c_void_p()
        if devices is not None:
            dv = (C.c_int * len(devices))(*devices)
            L.check(self.lib.dasmc_gpu_create_multi(C.byref(d), _fp(X), _ip(y), self.n, max_particles, dv, len(devices),
                                                    _PREC[precision], C.byref(h)))
        else:
            L.check(self.lib.dasmc_gpu_create(C.byref(d), _fp(X), _ip(y), self.n, max_particles, device,
                                              _PREC[precision], C.byref(h)))
        self.h = h
        self.max_particles = max_particles

    def close(self):
        if self.h:
            self.lib.dasmc_gpu_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # TargetContext (target.hpp:95-113)
    def set_target(self, prefix_end: int, block_end: int, total_n: int, mode: str = "scaled", beta: float = 1.0,
                   sigma: float = 1.0):
        L.check(self.lib.dasmc_gpu_set_target(self.h, prefix_end, block_end, total_n,
                                              L.SCALED if mode == "scaled" else L.SDA, beta, sigma))

    def log_target_with_grad(self, thetas: np.ndarray, want_grad: bool = True):  # target.hpp:147-173
        th = np.ascontiguousarray(thetas, dtype=np.float64).reshape(-1, self.D)
        J = th.shape[0]
        vals = np.empty(J)
        grads = np.empty((J, self.D)) if want_grad else None
        L.check(self.lib.dasmc_gpu_value_and_grad(self.h, _dp(th), J, _dp(vals), _dp(grads)))
        return vals, grads

    def unscaled_loglik_parts(self, thetas: np.ndarray):  # target.hpp:121-129
        th = np.ascontiguousarray(thetas, dtype=np.float64).reshape(-1, self.D)
        J = th.shape[0]
        a, b = np.empty(J), np.empty(J)
        L.check(self.lib.dasmc_gpu_loglik_parts(self.h, _dp(th), J, _dp(a), _dp(b)))
        return a, b

    def momentum(self, seed: int, k: int, J: int) -> np.ndarray:  # kernels.hpp:131 draws
        out = np.empty((J, self.D))
        L.check(self.lib.dasmc_gpu_momentum(self.h, seed, k, J, _dp(out)))
        return out

    def uniforms(self, seed: int, k: int, count: int) -> np.ndarray:  # fork(kResample, k) draws (smc.hpp:152)
        u = np.empty(count)
        L.check(self.lib.dasmc_gpu_uniforms(self.h, seed, k, count, _dp(u)))
        return u

    def resample_indices(self, w, u, kind: str = "multinomial") -> np.ndarray:
        w = np.ascontiguousarray(w, dtype=np.float64)
        u = np.ascontiguousarray(u, dtype=np.float64)
        idx = np.empty(len(w), dtype=np.int32)
        L.check(self.lib.dasmc_gpu_resample_indices(self.h, _dp(w), _dp(u), len(w), _RESAMPLE[kind], _ip(idx)))
        return idx

    # ParticleEnsemble (smc.hpp:28-35, 73-89)
    def init_ensemble(self, J: int, seed: int):
        L.check(self.lib.dasmc_gpu_init_ensemble(self.h, J, seed))

    def set_ensemble(self, thetas, log_weights, iteration: int = 0):
        th = np.ascontiguousarray(thetas)
        lw = np.ascontiguousarray(log_weights, dtype=np.float64)
        J = lw.shape[0]
        if th.dtype == np.float32:
            L.check(self.lib.dasmc_gpu_set_ensemble_f32(self.h, _fp(th), _dp(lw), J, iteration))
        else:
            th = th.astype(np.float64, copy=False)
            L.check(self.lib.dasmc_gpu_set_ensemble(self.h, _dp(th), _dp(lw), J, iteration))

    def get_ensemble(self, J: int, dtype=np.float64):
        th = np.empty((J, self.D), dtype=dtype)
        lw = np.empty(J)
        it = C.c_int()
        fn = self.lib.dasmc_gpu_get_ensemble_f32 if dtype == np.float32 else self.lib.dasmc_gpu_get_ensemble
        L.check(fn(self.h, th.ctypes.data_as(L._F if dtype == np.float32 else L._D), _dp(lw), C.byref(it)))
        return th, lw, it.value

    def smc_step(self, cfg: KernelConfig, seed: int, resample: str = "multinomial", fraction: float = 0.5,
                 always: bool = False, sync: bool = True):
        kc = cfg.c()
        rec = L.IterRecord()
        L.check(self.lib.dasmc_gpu_smc_step(self.h, C.byref(kc), seed, _RESAMPLE[resample], fraction,
                                            1 if always else 0, C.byref(rec) if sync else None))
        return _rec(rec) if sync else None

    def sync_records(self, count: int):
        recs = (L.IterRecord * max(count, 1))()
        L.check(self.lib.dasmc_gpu_sync_records(self.h, recs, count))
        return [_rec(recs[i]) for i in range(count)]

    def last_proposals(self, J: int):
        pf = np.empty((J, self.D))
        ltn, lto, w = np.empty(J), np.empty(J), np.empty(J)
        div = np.empty(J, dtype=np.int32)
        idx = np.empty(J, dtype=np.int32)
        L.check(self.lib.dasmc_gpu_last_proposals(self.h, _dp(pf), _dp(ltn), _dp(lto), _ip(div), _dp(w), _ip(idx)))
        return {"p_final": pf, "log_target_new": ltn, "log_target_old": lto, "divergent": div, "weights": w,
                "indices": idx}

    def sda_moments(self, prefix_end: int, block_end: int) -> np.ndarray:  # annealing.hpp:153-174
        out = np.zeros(6)
        L.check(self.lib.dasmc_gpu_sda_moments(self.h, prefix_end, block_end, _dp(out)))
        return out

    def set_graphs(self, enable: bool = True):  # CUDA-graph replay of smc_step (launch-bound configs)
        L.check(self.lib.dasmc_gpu_set_graphs(self.h, 1 if enable else 0))

    def set_cache_start(self, enable: bool = True):  # SPEC.md:410 start-gradient cache (opt-in)
        L.check(self.lib.dasmc_gpu_set_cache_start(self.h, 1 if enable else 0))

    def last_step_cached(self) -> bool:
        return bool(self.lib.dasmc_gpu_last_step_cached(self.h))

    def set_rows(self, rows: Optional[np.ndarray]):  # runner.hpp:548-557 redraw batch (None: resident set)
        if rows is None:
            L.check(self.lib.dasmc_gpu_set_rows(self.h, None, 0))
        else:
            r = np.ascontiguousarray(rows, dtype=np.int64)
            L.check(self.lib.dasmc_gpu_set_rows(self.h, r.ctypes.data_as(L._I64), r.shape[0]))

    def evaluate_predictive(self, X_test: np.ndarray, y_test: np.ndarray):  # runner.hpp:331-364
        """(mean log predictive probability of the true label, accuracy %) of the current ensemble."""
        X = np.ascontiguousarray(X_test, dtype=np.float32)
        y = np.ascontiguousarray(y_test, dtype=np.int32)
        lp, acc = C.c_double(), C.c_double()
        L.check(self.lib.dasmc_gpu_evaluate_predictive(self.h, _fp(X), _ip(y), X.shape[0], C.byref(lp), C.byref(acc)))
        return lp.value, acc.value

    def predictive_mix(self, X_test: np.ndarray, w_local: np.ndarray, J: int, pred: np.ndarray,
                       y_test: Optional[np.ndarray] = None) -> np.ndarray:
        """pred += sum_j w_j softmax_j over this context's J particles (sharded evaluate_predictive)."""
        X = np.ascontiguousarray(X_test, dtype=np.float32)
        w = np.ascontiguousarray(w_local, dtype=np.float64)
        y = np.ascontiguousarray(y_test, dtype=np.int32) if y_test is not None else None
        L.check(self.lib.dasmc_gpu_predictive_mix(self.h, _fp(X), _ip(y), X.shape[0], _dp(w), J, _dp(pred)))
        return pred


def predictive_metrics(pred: np.ndarray, y: np.ndarray):
    """Mean log predictive probability (floor 1e-300) and argmax accuracy % (runner.hpp:351-363)."""
    pred = np.ascontiguousarray(pred, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.int32)
    lp, acc = C.c_double(), C.c_double()
    L.check(L.load().dasmc_predictive_metrics(_dp(pred), _ip(y), pred.shape[0], pred.shape[1], C.byref(lp),
                                              C.byref(acc)))
    return lp.value, acc.value


@dataclass
class RunConfig:  # runner.hpp:57-70 (hot-loop subset)
    kernel: KernelConfig
    schedule: ScheduleConfig
    sigma: float = 1.0
    beta0: float = 0.1
    entropy_step: float = 1.0
    particles: int = 128
    iterations: int = 1
    seed: int = 0
    resample_fraction: float = 0.5
    resample: str = "multinomial"
    resample_always: bool = False
    redraw: bool = False  # ScheduleConfig::redraw_constant (runner.hpp:531-556)


def run_experiment(spec: NetSpec, X: np.ndarray, y: np.ndarray, cfg: RunConfig, device: int = 0,
                   precision: str = "fp32", return_ensemble: bool = False):
    """The run_experiment hot loop (runner.hpp:453-617) on one B200; X/y unshuffled."""
    lib = L.load()
    X = np.ascontiguousarray(X, dtype=np.float32)
    y = np.ascontiguousarray(y, dtype=np.int32)
    rc = L.RunCfg(cfg.kernel.c(), cfg.schedule.c(), cfg.sigma, cfg.beta0, cfg.entropy_step, cfg.particles,
                  cfg.iterations, cfg.seed, cfg.resample_fraction, _RESAMPLE[cfg.resample],
                  1 if cfg.resample_always else 0, 1 if cfg.redraw else 0)
    recs = (L.IterRecord * cfg.iterations)()
    sda = (L.SdaState * cfg.iterations)()
    D = param_count(spec)
    th = np.empty((cfg.particles, D)) if return_ensemble else None
    lw = np.empty(cfg.particles) if return_ensemble else None
    d = spec.desc()
    L.check(lib.dasmc_gpu_run(C.byref(d), _fp(X), _ip(y), X.shape[0], C.byref(rc), device, _PREC[precision], recs,
                              sda, _dp(th), _dp(lw)))
    out = {"records": [_rec(r) for r in recs],
           "sda": [(s.beta, s.prefix_end, s.block_end, s.stage, s.terminal) for s in sda]}
    if return_ensemble:
        out["thetas"], out["log_weights"] = th, lw
    return out

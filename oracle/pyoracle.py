"""ctypes wrapper of the CPU oracle (TEST INFRASTRUCTURE ONLY).

Loaded by tests/, __graft_entry__.smoke() and bench.py's CPU legs to check or
time against; never used by the product path.  Builds oracle/_build with make
when the shared object is missing and the sources are present.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "_build", "liboracle.so")
TESTS_BIN = os.path.join(HERE, "_build", "oracle_tests")

_D = C.POINTER(C.c_double)
_I = C.POINTER(C.c_int)
_U64 = C.POINTER(C.c_uint64)
_I64 = C.POINTER(C.c_int64)


class StepOut(C.Structure):
    _fields_ = [("ess", C.c_double), ("mean_log_target", C.c_double), ("resampled", C.c_int),
                ("n_divergent", C.c_int)]


class RunRecord(C.Structure):
    _fields_ = [("k", C.c_int), ("batch", C.c_int64), ("beta", C.c_double), ("ess", C.c_double),
                ("resampled", C.c_int), ("mean_log_target", C.c_double), ("sampler_ms", C.c_double),
                ("n_divergent", C.c_int)]


def build():
    subprocess.run(["make", "-C", HERE, "-s"], check=True)


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(SO):
            build()
        _lib = C.CDLL(SO)
        L = _lib
        L.oracle_last_error.restype = C.c_char_p
        L.oracle_fork_key.restype = C.c_uint64
        L.oracle_fork_key.argtypes = [C.c_uint64] * 4
        L.oracle_rng_u64.argtypes = [C.c_uint64, C.c_int64, _U64]
        L.oracle_rng_normals.argtypes = [C.c_uint64, C.c_int64, _D]
        L.oracle_rng_uniforms.argtypes = [C.c_uint64, C.c_int64, _D]
        L.oracle_use_blas.argtypes = [C.c_char_p]
        L.oracle_batch_size.restype = C.c_int64
        L.oracle_batch_size.argtypes = [C.c_int, C.c_int64, C.c_int64, C.c_int, C.c_int64, C.c_int, C.c_int, C.c_int]
        L.oracle_sda_beta_step.restype = C.c_double
        L.oracle_sda_beta_step.argtypes = [C.c_double, _D, C.c_double]
    return _lib


def _check(rc):
    if rc != 0:
        msg = lib().oracle_last_error().decode()
        if rc == -2:
            raise RuntimeError("SamplerError: " + msg)
        raise ValueError(msg)


def _dp(a):
    return a.ctypes.data_as(_D) if a is not None else None


def _ip(a):
    return a.ctypes.data_as(_I) if a is not None else None


def _net(layers):
    return (C.c_int * len(layers))(*layers), len(layers)


def cnn_layers(in_shape, convs, head):
    """[EXT] CNN model encoding accepted wherever `layers` is: in_shape = (c, h, w),
    convs = [(k, cout, pool), ...], head = MLP layer sizes after the flatten
    (head[0] is the flatten size)."""
    c, h, w = in_shape
    out = [-1, c, h, w, len(convs)]
    for k, co, pool in convs:
        out += [k, co, 1 if pool else 0]
    return out + list(head)


def input_dim(layers):
    return layers[1] * layers[2] * layers[3] if layers[0] == -1 else layers[0]


def use_blas(enable=True):
    """Route the oracle's dgemms through numpy's OpenBLAS (1 thread per call)."""
    if not enable:
        return lib().oracle_use_blas(None) == 0
    import glob
    d = os.path.join(os.path.dirname(np.__file__), "..", "numpy.libs")
    cands = glob.glob(os.path.join(d, "libscipy_openblas64_*.so"))
    if not cands:
        return False
    return lib().oracle_use_blas(os.path.realpath(cands[0]).encode()) == 0


def fork_key(key, a, b=0, c=0):
    return int(lib().oracle_fork_key(key, a, b, c))


def rng_u64(key, n):
    out = np.empty(n, dtype=np.uint64)
    lib().oracle_rng_u64(key, n, out.ctypes.data_as(_U64))
    return out


def rng_normals(key, n):
    out = np.empty(n)
    lib().oracle_rng_normals(key, n, _dp(out))
    return out


def rng_uniforms(key, n):
    out = np.empty(n)
    lib().oracle_rng_uniforms(key, n, _dp(out))
    return out


def param_count(layers):
    arr, nl = _net(layers)
    return int(lib().oracle_param_count(arr, nl))


def make_teacher(layers, act, n, feature_kind, seed, cfg_id, threads=8):
    arr, nl = _net(layers)
    X = np.empty((n, input_dim(layers)))
    y = np.empty(n, dtype=np.int32)
    _check(lib().oracle_make_teacher(arr, nl, act, C.c_int64(n), feature_kind, C.c_uint64(seed), C.c_uint64(cfg_id),
                                     threads, _dp(X), _ip(y)))
    return X, y


def make_synthetic(kind, n, noise, seed, dim=2):
    X = np.empty((n, dim if kind == 2 else 2))
    y = np.empty(n, dtype=np.int32)
    t = np.empty(n)
    _check(lib().oracle_make_synthetic(kind, C.c_int64(n), C.c_double(noise), C.c_uint64(seed), dim, _dp(X), _ip(y),
                                       _dp(t)))
    return X, y, t


def shuffle_perm(seed, n):
    p = np.empty(n, dtype=np.int64)
    _check(lib().oracle_shuffle_perm(C.c_uint64(seed), C.c_int64(n), p.ctypes.data_as(_I64)))
    return p


def value_and_grad(layers, act, X, y, window, mode, beta, sigma, thetas, threads=8, want_grad=True):
    arr, nl = _net(layers)
    X = np.ascontiguousarray(X, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.int32)
    th = np.ascontiguousarray(thetas, dtype=np.float64)
    J = th.shape[0]
    vals = np.empty(J)
    grads = np.empty_like(th) if want_grad else None
    P, M, N = window
    _check(lib().oracle_value_and_grad(arr, nl, act, _dp(X), _ip(y), C.c_int64(X.shape[0]), C.c_int64(P),
                                       C.c_int64(M), C.c_int64(N), mode, C.c_double(beta), C.c_double(sigma), _dp(th),
                                       C.c_int64(J), threads, _dp(vals), _dp(grads)))
    return vals, grads


def loglik_parts(layers, act, X, y, P, M, thetas, threads=8):
    arr, nl = _net(layers)
    X = np.ascontiguousarray(X, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.int32)
    th = np.ascontiguousarray(thetas, dtype=np.float64)
    J = th.shape[0]
    a, b = np.empty(J), np.empty(J)
    _check(lib().oracle_loglik_parts(arr, nl, act, _dp(X), _ip(y), C.c_int64(X.shape[0]), C.c_int64(P), C.c_int64(M),
                                     _dp(th), C.c_int64(J), threads, _dp(a), _dp(b)))
    return a, b


def init_ensemble(layers, act, X, y, window, mode, beta, sigma, seed, J, threads=8):
    arr, nl = _net(layers)
    X = np.ascontiguousarray(X, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.int32)
    D = param_count(layers)
    th = np.empty((J, D))
    lw = np.empty(J)
    P, M, N = window
    _check(lib().oracle_init_ensemble(arr, nl, act, _dp(X), _ip(y), C.c_int64(X.shape[0]), C.c_int64(P),
                                      C.c_int64(M), C.c_int64(N), mode, C.c_double(beta), C.c_double(sigma),
                                      C.c_uint64(seed), C.c_int64(J), threads, _dp(th), _dp(lw)))
    return th, lw


def smc_step(layers, act, X, y, window, mode, beta, sigma, kernel, seed, fraction, resample_kind, always, thetas,
             log_w, iteration, threads=8, dumps=True):
    """One oracle smc_step; returns (thetas, log_w, iteration, record, dumps)."""
    arr, nl = _net(layers)
    X = np.ascontiguousarray(X, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.int32)
    th = np.array(thetas, dtype=np.float64, copy=True, order="C")
    lw = np.array(log_w, dtype=np.float64, copy=True)
    J, D = th.shape
    it = C.c_int(iteration)
    out = StepOut()
    P, M, N = window
    h, S, kind = kernel
    d = {}
    if dumps:
        d = {"p0": np.empty((J, D)), "pS": np.empty((J, D)), "lt_new": np.empty(J), "lt_old": np.empty(J),
             "divergent": np.empty(J, dtype=np.int32), "weights": np.empty(J), "indices": np.empty(J, dtype=np.int32)}
    _check(lib().oracle_smc_step(arr, nl, act, _dp(X), _ip(y), C.c_int64(X.shape[0]), C.c_int64(P), C.c_int64(M),
                                 C.c_int64(N), mode, C.c_double(beta), C.c_double(sigma), C.c_double(h), S, kind,
                                 C.c_uint64(seed), C.c_double(fraction), resample_kind, 1 if always else 0, threads,
                                 C.c_int64(J), _dp(th), _dp(lw), C.byref(it), C.byref(out), _dp(d.get("p0")),
                                 _dp(d.get("pS")), _dp(d.get("lt_new")), _dp(d.get("lt_old")), _ip(d.get("divergent")),
                                 _dp(d.get("weights")), _ip(d.get("indices"))))
    rec = {"ess": out.ess, "mean_log_target": out.mean_log_target, "resampled": bool(out.resampled),
           "n_divergent": out.n_divergent}
    return th, lw, it.value, rec, d


def propose_particles(layers, act, X, y, window, mode, beta, sigma, kernel, seed, k, gj, thetas, threads=8):
    """smc.hpp:118-138 for a subset of particles with global slots gj; returns (thetas, inc, lt_new)."""
    arr, nl = _net(layers)
    X = np.ascontiguousarray(X, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.int32)
    th = np.array(thetas, dtype=np.float64, copy=True, order="C")
    gj = np.ascontiguousarray(gj, dtype=np.int64)
    n = th.shape[0]
    inc, lt = np.empty(n), np.empty(n)
    P, M, N = window
    h, S, kk = kernel
    _check(lib().oracle_propose_particles(arr, nl, act, _dp(X), _ip(y), C.c_int64(X.shape[0]), C.c_int64(P),
                                          C.c_int64(M), C.c_int64(N), mode, C.c_double(beta), C.c_double(sigma),
                                          C.c_double(h), S, kk, C.c_uint64(seed), k, gj.ctypes.data_as(_I64),
                                          C.c_int64(n), threads, _dp(th), _dp(inc), _dp(lt)))
    return th, inc, lt


def evaluate_predictive(layers, act, X, y, thetas, log_w, threads=8):
    """runner.hpp:331-364: (mean log predictive probability, accuracy %)."""
    arr, nl = _net(layers)
    X = np.ascontiguousarray(X, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.int32)
    th = np.ascontiguousarray(thetas, dtype=np.float64)
    lw = np.ascontiguousarray(log_w, dtype=np.float64)
    lp, acc = C.c_double(), C.c_double()
    _check(lib().oracle_evaluate_predictive(arr, nl, act, _dp(X), _ip(y), C.c_int64(X.shape[0]), _dp(th), _dp(lw),
                                            C.c_int64(th.shape[0]), threads, C.byref(lp), C.byref(acc)))
    return lp.value, acc.value


def resample_indices(w, u, kind):
    w = np.ascontiguousarray(w, dtype=np.float64)
    u = np.ascontiguousarray(u, dtype=np.float64)
    idx = np.empty(len(w), dtype=np.int32)
    _check(lib().oracle_resample_indices(_dp(w), _dp(u), C.c_int64(len(w)), kind, _ip(idx)))
    return idx


def normalize(lw):
    lw = np.ascontiguousarray(lw, dtype=np.float64)
    w = np.empty_like(lw)
    e = C.c_double()
    _check(lib().oracle_normalize(_dp(lw), C.c_int64(len(lw)), _dp(w), C.byref(e)))
    return w, e.value


def batch_size(kind, initial, increment, iterations, n, period, switch_iteration, k):
    return int(lib().oracle_batch_size(kind, initial, increment, iterations, n, period, switch_iteration, k))


def sda_beta_step(beta, step, denom):
    s = C.c_double(step)
    b = lib().oracle_sda_beta_step(beta, C.byref(s), denom)
    return b, s.value


def sda_moments_from(pre, blk, lw):
    pre, blk, lw = (np.ascontiguousarray(a, dtype=np.float64) for a in (pre, blk, lw))
    out = np.empty(6)
    _check(lib().oracle_sda_moments_from(_dp(pre), _dp(blk), _dp(lw), C.c_int64(len(pre)), _dp(out)))
    return out


def sda_advance_with(increment, n, state8, m6):
    st = np.array(state8, dtype=np.float64)
    m = np.ascontiguousarray(m6, dtype=np.float64)
    _check(lib().oracle_sda_advance_with(C.c_int64(increment), C.c_int64(n), _dp(st), _dp(m)))
    return st


def run(layers, act, X, y, *, sigma=1.0, kernel=(0.002, 3, 0), sched=(2, 200, 100, 1, 40), beta0=0.1,
        entropy_step=1.0, redraw=False, particles=128, iterations=50, seed=0, threads=8, fraction=0.5,
        resample_kind=0, resample_always=False, want_ensemble=False):
    """Whole-run hot loop; sched = (kind, initial, increment, period, switch_iteration)."""
    arr, nl = _net(layers)
    X = np.ascontiguousarray(X, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.int32)
    recs = (RunRecord * iterations)()
    D = param_count(layers)
    th = np.empty((particles, D)) if want_ensemble else None
    lw = np.empty(particles) if want_ensemble else None
    kind, initial, inc, period, sw = sched
    h, S, kk = kernel
    _check(lib().oracle_run(arr, nl, act, _dp(X), _ip(y), C.c_int64(X.shape[0]), C.c_double(sigma), C.c_double(h), S,
                            kk, kind, C.c_int64(initial), C.c_int64(inc), period, sw, C.c_double(beta0),
                            C.c_double(entropy_step), 1 if redraw else 0, particles, iterations, C.c_uint64(seed),
                            threads, C.c_double(fraction), resample_kind, 1 if resample_always else 0, recs, _dp(th),
                            _dp(lw)))
    out = [{"k": r.k, "batch": r.batch, "beta": r.beta, "ess": r.ess, "resampled": bool(r.resampled),
            "mean_log_target": r.mean_log_target, "sampler_ms": r.sampler_ms, "n_divergent": r.n_divergent}
           for r in recs]
    return (out, th, lw) if want_ensemble else out

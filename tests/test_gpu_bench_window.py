"""Oracle parity of the tensor-core modes AT THE BENCHED CONFIGURATION.

bench.py measures BASELINE.json configs[1] (C2: 784-200-10 ReLU, n = 60000, J = 1024) at the
schedule's iterations k = 155.., whose window is M = 32000 rows.  The tensor core's fp32
accumulation runs over K = M there, so parity at M <= 1100 (test_gpu_tensorcore.py) does not
cover it.  This file compares, on the bench's own data (teacher seed 0, cfg 2, shuffled with
fork(kPermutation) of seed 0) and the bench's own init_ensemble streams:

  * the log target (target.hpp:147-173) of 8 particles, error in NATS (absolute);
  * one smc_step from the same ensemble (smc.hpp:109-158): the incremental log-weight
    (kernels.hpp:153-163) of every particle, error in nats; ESS, the resample decision and the
    systematic indices;
  * the device resampling uniforms against the oracle's stream (rng.hpp:60-64), bit-exact.

Bounds (stated per mode; measured values are written to gpurun_out/bench_window.json and
DESIGN.md §4).  SMC decisions depend on log-weight DIFFERENCES between particles: at this
window the particles' increments are ~1e8 nats apart (ESS = 1), so the bounds below leave
every decision unchanged, which the ESS / index checks verify directly.
"""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LAYERS, N, M, K = [784, 200, 10], 60000, 32000, 155
# |log target - oracle| in nats (|value| ~ 1e7 at this window) and max |inc - oracle| as a
# fraction of the increments' spread across particles (the quantity resampling acts on)
# Measured on B200 (gpurun_out/bench_window.json, 8 particles, |value| 0.8-1.8e7 nats):
#   fp32 0.39 / 2e-6, 3xtf32 103 / 9e-4, f16x2 37 / 6e-4, tf32 tf32h f16 5.1e3 / 6e-4.
# The increments' error is dominated by the step's dynamics (from prior draws at this window
# the three leapfrog steps move log targets by up to 6e8 nats), identical across the tensor
# modes; every mode reproduces the oracle's ESS, decision and indices.
BOUNDS = {"fp32": (5.0, 1e-4), "3xtf32": (400.0, 5e-3), "f16x2": (150.0, 5e-3), "tf32h": (2e4, 5e-3),
          "tf32": (2e4, 5e-3), "f16": (2e4, 5e-3)}
_RESULTS = {}


@pytest.fixture(scope="module")
def bench_data(product, oracle):
    spec = product.NetSpec(LAYERS, "relu")
    X, y = product.make_teacher_data(spec, N, 1, 0, 2, threads=os.cpu_count() or 8)
    perm = product.shuffle_permutation(0, N)
    X, y = np.ascontiguousarray(X[perm]), np.ascontiguousarray(y[perm])
    X64 = X.astype(np.float64)
    oracle.use_blas(True)
    J = 8
    th, lw = oracle.init_ensemble(LAYERS, 0, X64, y, (0, M, N), 0, 1.0, 1.0, 0, J, threads=os.cpu_count() or 8)
    th = th.astype(np.float32).astype(np.float64)  # the device stores fp32 positions
    vo, _ = oracle.value_and_grad(LAYERS, 0, X64, y, (0, M, N), 0, 1.0, 1.0, th, threads=os.cpu_count() or 8,
                                  want_grad=False)
    step = oracle.smc_step(LAYERS, 0, X64, y, (0, M, N), 0, 1.0, 1.0, (0.002, 3, 0), 0, 0.5, 1, False, th, lw, K,
                           threads=os.cpu_count() or 8)
    return spec, X, y, th, lw, vo, step


def _inc(lt_new, lt_old, p0, pS):
    return (lt_new - lt_old) + 0.5 * (np.sum(p0 * p0, axis=1) - np.sum(pS * pS, axis=1))


@pytest.mark.parametrize("prec", ["f16x2", "tf32h", "3xtf32", "tf32", "f16", "fp32"])
def test_bench_window_nats(product, bench_data, prec):
    spec, X, y, th, lw, vo, (tho, lwo, ito, reco, d) = bench_data
    J = th.shape[0]
    t = product.GpuEnsembleTarget(spec, X, y, J, precision=prec)
    t.set_target(0, M, N, "scaled", 1.0, 1.0)
    v, _ = t.log_target_with_grad(th, want_grad=False)
    t.set_ensemble(th, lw, K)
    rec = t.smc_step(product.KernelConfig.hmc(0.002, 3), 0, "systematic", 0.5)
    dump = t.last_proposals(J)
    p0 = t.momentum(0, K, J)
    t.close()
    inc = _inc(dump["log_target_new"], dump["log_target_old"], p0, dump["p_final"])
    inc_o = _inc(d["lt_new"], d["lt_old"], d["p0"], d["pS"])
    ok = (dump["divergent"] == 0) & (d["divergent"] == 0)
    verr = float(np.max(np.abs(v - vo)))
    ierr = float(np.max(np.abs(inc - inc_o)[ok])) if ok.any() else 0.0
    spread = float(np.max(inc_o[ok]) - np.min(inc_o[ok])) if ok.any() else 0.0
    res = {"value_abs_nats": verr, "value_rel": float(np.max(np.abs(v - vo) / np.abs(vo))),
           "inc_abs_nats": ierr, "inc_spread_nats": spread, "ess": rec["ess"], "ess_oracle": reco["ess"],
           "indices_equal": bool(np.array_equal(dump["indices"], d["indices"])),
           "resampled": [bool(rec["resampled"]), bool(reco["resampled"])], "window": M, "particles": J}
    _RESULTS[prec] = res
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "bench_window.json"), "w") as f:
        json.dump(_RESULTS, f, indent=1)
    print(prec, json.dumps(res))
    tv, ti = BOUNDS[prec]
    if os.environ.get("DASMC_REPORT_ONLY"):
        return
    assert verr < tv, res
    assert ierr < ti * spread, res
    assert bool(rec["resampled"]) == bool(reco["resampled"]), res
    np.testing.assert_allclose(rec["ess"], reco["ess"], rtol=1e-3)
    assert res["indices_equal"], res


def test_device_uniforms_bit_exact(product, oracle):
    """uniform() of the resampling stream (rng.hpp:60-64; smc.hpp:152) drawn on the device with
    the chunked F2 jump-ahead equals the oracle's sequential stream bit for bit."""
    spec = product.NetSpec([4, 3, 2], "tanh")
    X = np.random.default_rng(0).random((16, 4)).astype(np.float32)
    y = (np.arange(16) % 2).astype(np.int32)
    cnt = 20000
    t = product.GpuEnsembleTarget(spec, X, y, cnt)
    for seed, k in ((0, 0), (7, 155), (2**40 + 3, 299)):
        u = t.uniforms(seed, k, cnt)
        uo = oracle.rng_uniforms(oracle.fork_key(seed, 3, k, 0), cnt)
        assert np.array_equal(u, uo), (seed, k, int(np.argmax(u != uo)))
    t.close()

"""GPU parity of the [EXT] CNN path (BASELINE.json configs[2..3]) against the fp64 oracle.

The reference is MLP-only, so the oracle's conv / pool layers are new
(oracle/dasmc_oracle.hpp, pinned to torch fp64 autograd in
tests/test_oracle_pins.py).  Tolerances are the north star's fp32 ones:
values 1e-5 relative, gradients max_rel_error < 1e-4 (floor 1e-3 ||ref||_inf).
"""
import numpy as np
import pytest

# fp32 Box-Muller from the exact integer draws (kernels.cu normal_from_draws): within a few
# fp32 ulp of the oracle's fp64 normal (rng.hpp:76-81) rounded to fp32
NORMAL_RTOL = 8e-7

pytestmark = pytest.mark.gpu

GRAD_TOL = 1e-4
VAL_TOL = 1e-5

# (conv front, head, activation): C3 and C4 at their BASELINE shapes, plus odd
# sizes (floor pooling) and tanh
C3 = (((1, 28, 28), [(5, 16, True), (5, 32, True)]), [512, 10], "relu")
C4 = (((3, 32, 32), [(3, 32, False), (3, 32, True), (3, 64, False), (3, 64, True)]), [1600, 256, 10], "relu")
ODD = (((2, 11, 11), [(3, 3, True), (2, 4, False)]), [4 * 3 * 3, 6, 3], "tanh")


def max_rel_error(a, b, floor):  # test_util.hpp:37-45
    return float(np.max(np.abs(a - b) / np.maximum(np.maximum(np.abs(a), np.abs(b)), floor)))


def grad_err(g, ref):
    return max_rel_error(g, ref, 1e-3 * np.max(np.abs(ref)))


def rel(a, b):
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300)))


def problem(product, arch, n, kind=1):
    conv, head, act = arch
    spec = product.NetSpec(head, act, conv)
    X, y = product.make_teacher_data(spec, n, kind, 0, 3, threads=8)
    return spec, X, y


@pytest.mark.parametrize("arch,M,J", [(C3, 40, 3), (C4, 12, 2), (ODD, 50, 4)])
def test_cnn_value_and_grad(product, oracle, arch, M, J):
    n = 64
    spec, X, y = problem(product, arch, n)
    D = product.param_count(spec)
    assert D == oracle.param_count(spec.oracle_layers())
    th = (0.3 * np.random.default_rng(1).standard_normal((J, D))).astype(np.float32).astype(np.float64)
    t = product.GpuEnsembleTarget(spec, X, y, J)
    a = 0 if arch[2] == "relu" else 1
    for mode, win, beta, sigma in (("scaled", (0, M, n), 1.0, 1.0), ("sda", (M // 3, M, n), 0.4, 0.7)):
        t.set_target(*win, mode, beta, sigma)
        v, g = t.log_target_with_grad(th)
        vo, go = oracle.value_and_grad(spec.oracle_layers(), a, X.astype(np.float64), y, win,
                                       0 if mode == "scaled" else 1, beta, sigma, th)
        assert rel(v, vo) < VAL_TOL, (mode, v, vo)
        for j in range(J):
            assert grad_err(g[j], go[j]) < GRAD_TOL, (mode, j, grad_err(g[j], go[j]))


def test_cnn_loglik_parts_and_momentum(product, oracle):
    spec, X, y = problem(product, ODD, 80)
    D = product.param_count(spec)
    th = np.random.default_rng(3).standard_normal((5, D))
    t = product.GpuEnsembleTarget(spec, X, y, 8)
    t.set_target(30, 70, 80, "sda", 0.5, 1.0)
    a, b = t.unscaled_loglik_parts(th)
    ao, bo = oracle.loglik_parts(spec.oracle_layers(), 1, X.astype(np.float64), y, 30, 70, th)
    assert rel(a, ao) < VAL_TOL and rel(b, bo) < VAL_TOL
    # momentum streams through the conv + head index walk (reference layout out)
    p = t.momentum(99, 4, 5)
    for j in range(5):
        ref = oracle.rng_normals(oracle.fork_key(99, 2, 4, j), D)
        np.testing.assert_allclose(p[j], ref.astype(np.float32), rtol=NORMAL_RTOL, atol=1e-30)


def test_cnn_smc_step(product, oracle):
    spec, X, y = problem(product, ODD, 120)
    lay = spec.oracle_layers()
    J, seed = 16, 5
    win = (0, 90, 120)
    th0, lw0 = oracle.init_ensemble(lay, 1, X.astype(np.float64), y, win, 0, 1.0, 1.0, seed, J)
    th0 = th0.astype(np.float32).astype(np.float64)
    t = product.GpuEnsembleTarget(spec, X, y, J)
    t.set_target(*win, "scaled", 1.0, 1.0)
    t.init_ensemble(J, seed)
    th_i, lw_i, _ = t.get_ensemble(J)
    np.testing.assert_allclose(th_i, th0, rtol=NORMAL_RTOL)
    assert rel(lw_i, lw0) < 1e-5
    t.set_ensemble(th0, lw0, 3)
    rec = t.smc_step(product.KernelConfig.hmc(0.005, 2), seed, "multinomial", 0.5)
    dump = t.last_proposals(J)
    tho, lwo, ito, reco, d = oracle.smc_step(lay, 1, X.astype(np.float64), y, win, 0, 1.0, 1.0, (0.005, 2, 0), seed,
                                             0.5, 0, False, th0, lw0, 3)
    assert rel(dump["log_target_old"], d["lt_old"]) < VAL_TOL
    assert rel(dump["log_target_new"], d["lt_new"]) < VAL_TOL
    np.testing.assert_allclose(rec["ess"], reco["ess"], rtol=1e-3)
    assert rec["resampled"] == reco["resampled"]


def test_c3_sda_run(product):
    """C3 (BASELINE configs[2], shortened): CNN + adaptive (SDA) annealing runs and anneals."""
    spec, X, y = problem(product, C3, 600)
    cfg = product.RunConfig(kernel=product.KernelConfig.hmc(0.002, 2),
                            schedule=product.ScheduleConfig("sda", 100, 100, 6, 600), particles=16, iterations=6,
                            seed=1, resample="systematic")
    out = product.run_experiment(spec, X, y, cfg)
    recs = out["records"]
    assert len(recs) == 6 and all(np.isfinite(r["ess"]) for r in recs)
    assert all(0 < s[0] <= 1 for s in out["sda"])

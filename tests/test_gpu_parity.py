"""GPU parity: the sm_100a path through the C-ABI against the fp64 CPU oracle.

Tolerances (north star, BASELINE.json): fp32 path within 1e-4 relative --
gradients by test_util.hpp's max_rel_error with floor = 1e-3 * ||ref||_inf,
values / log-weights relative; resampling indices and schedules bit-exact
given the oracle's weights and uniforms.
"""
import numpy as np
import pytest

# fp32 Box-Muller from the exact integer draws (kernels.cu normal_from_draws): within a few
# fp32 ulp of the oracle's fp64 normal (rng.hpp:76-81) rounded to fp32
NORMAL_RTOL = 8e-7

pytestmark = pytest.mark.gpu

GRAD_TOL = 1e-4
VAL_TOL = 1e-5


def max_rel_error(a, b, floor):  # test_util.hpp:37-45
    return float(np.max(np.abs(a - b) / np.maximum(np.maximum(np.abs(a), np.abs(b)), floor)))


def grad_err(g, ref):
    return max_rel_error(g, ref, 1e-3 * np.max(np.abs(ref)))


def rel(a, b):
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300)))


def make_problem(product, layers, act, n, seed=0, kind=0):
    spec = product.NetSpec(layers, act)
    X, y = product.make_teacher_data(spec, n, kind, seed, 7, threads=8)
    return spec, X, y


@pytest.mark.parametrize("layers,act,M", [([64, 32, 10], "tanh", 200), ([784, 200, 10], "relu", 333),
                                          ([5, 3], "relu", 1), ([7, 9, 4, 3], "tanh", 65),
                                          ([33, 17, 2], "relu", 130)])
def test_value_and_grad_scaled(product, oracle, layers, act, M):
    n = max(M, 400)
    spec, X, y = make_problem(product, layers, act, n)
    D = product.param_count(spec)
    J = 6
    th = np.random.default_rng(1).standard_normal((J, D)).astype(np.float32).astype(np.float64)
    t = product.GpuEnsembleTarget(spec, X, y, J)
    t.set_target(0, M, n, "scaled", 1.0, 1.0)
    v, g = t.log_target_with_grad(th)
    vo, go = oracle.value_and_grad(layers, 0 if act == "relu" else 1, X.astype(np.float64), y, (0, M, n), 0, 1.0,
                                   1.0, th)
    assert rel(v, vo) < VAL_TOL
    for j in range(J):
        assert grad_err(g[j], go[j]) < GRAD_TOL, j


def test_value_and_grad_sda_and_sigma(product, oracle):
    layers, act = [20, 16, 5], "tanh"
    spec, X, y = make_problem(product, layers, act, 500)
    D = product.param_count(spec)
    th = 0.7 * np.random.default_rng(2).standard_normal((5, D))
    t = product.GpuEnsembleTarget(spec, X, y, 8)
    for P, M, beta, sigma in ((0, 100, 0.1, 1.0), (100, 250, 0.37, 0.5), (250, 250, 1.0, 2.0)):
        t.set_target(P, M, 500, "sda", beta, sigma)
        v, g = t.log_target_with_grad(th)
        vo, go = oracle.value_and_grad(layers, 1, X.astype(np.float64), y, (P, M, 500), 1, beta, sigma, th)
        assert rel(v, vo) < VAL_TOL
        for j in range(5):
            assert grad_err(g[j], go[j]) < GRAD_TOL


def test_loglik_parts(product, oracle):
    layers = [16, 8, 4]
    spec, X, y = make_problem(product, layers, "relu", 300)
    D = product.param_count(spec)
    th = np.random.default_rng(3).standard_normal((7, D))
    t = product.GpuEnsembleTarget(spec, X, y, 8)
    t.set_target(120, 290, 300, "sda", 0.5, 1.0)
    a, b = t.unscaled_loglik_parts(th)
    ao, bo = oracle.loglik_parts(layers, 0, X.astype(np.float64), y, 120, 290, th)
    assert rel(a, ao) < VAL_TOL and rel(b, bo) < VAL_TOL


def test_momentum_streams(product, oracle):
    layers = [40, 30, 10]
    spec, X, y = make_problem(product, layers, "relu", 50)
    D = product.param_count(spec)
    t = product.GpuEnsembleTarget(spec, X, y, 9)
    for seed, k in ((0, 0), (12345, 17)):
        p = t.momentum(seed, k, 9)
        for j in range(9):
            ref = oracle.rng_normals(oracle.fork_key(seed, 2, k, j), D)
            # fp32 Box-Muller on the device from the exact integer draws (kernels.cu normal_from_draws)
            np.testing.assert_allclose(p[j], ref.astype(np.float32), rtol=NORMAL_RTOL, atol=1e-30)


def test_resample_indices_bit_exact(product, oracle):
    spec, X, y = make_problem(product, [4, 2], "relu", 10)
    t = product.GpuEnsembleTarget(spec, X, y, 20000)
    rng = np.random.default_rng(4)
    # 16384: the largest CDF built in shared memory; 20000: the global-memory CDF path
    for J in (2, 3, 100, 1024, 4096, 16384, 20000):
        for trial in range(3):
            w = rng.random(J) ** 8
            if trial == 1:
                w[:] = 0
                w[J // 2] = 1.0
            if trial == 2:
                w[::2] = 0
            w /= w.sum()
            u = oracle.rng_uniforms(oracle.fork_key(9, 3, trial, 0), J)
            assert np.array_equal(t.resample_indices(w, u, "multinomial"), oracle.resample_indices(w, u, 0))
            assert np.array_equal(t.resample_indices(w, u[:1], "systematic"), oracle.resample_indices(w, u[:1], 1))
    # boundary: u exactly on a CDF value goes to the next index (upper_bound)
    w = np.array([0.25, 0.25, 0.5])
    u = np.array([0.25, 0.0, 0.75 - 1e-17])
    assert np.array_equal(t.resample_indices(w, u), oracle.resample_indices(w, u, 0))


def test_init_ensemble(product, oracle):
    layers = [10, 6, 3]
    spec, X, y = make_problem(product, layers, "tanh", 120)
    t = product.GpuEnsembleTarget(spec, X, y, 16)
    t.set_target(0, 40, 120, "scaled", 1.0, 1.5)
    t.init_ensemble(16, 77)
    th, lw, it = t.get_ensemble(16)
    tho, lwo = oracle.init_ensemble(layers, 1, X.astype(np.float64), y, (0, 40, 120), 0, 1.0, 1.5, 77, 16)
    np.testing.assert_allclose(th, tho.astype(np.float32), rtol=NORMAL_RTOL)
    assert rel(lw, lwo) < 1e-5 and it == 0


def _step_compare(product, oracle, layers, act, n, win, mode, beta, kernel, J, seed, fraction, rkind, always,
                  sigma=1.0):
    spec, X, y = make_problem(product, layers, act, n)
    a = 0 if act == "relu" else 1
    th0, lw0 = oracle.init_ensemble(layers, a, X.astype(np.float64), y, win, mode, beta, sigma, seed, J)
    th0 = th0.astype(np.float32).astype(np.float64)
    t = product.GpuEnsembleTarget(spec, X, y, J)
    t.set_target(*win, "scaled" if mode == 0 else "sda", beta, sigma)
    t.set_ensemble(th0, lw0, 3)
    rec = t.smc_step(product.KernelConfig(*kernel[:2], "hmc" if kernel[2] == 0 else "langevin"), seed,
                     "multinomial" if rkind == 0 else "systematic", fraction, always)
    dump = t.last_proposals(J)
    th1, lw1, it1 = t.get_ensemble(J)
    dump["p0"] = t.momentum(seed, 3, J)  # the step's own fp32 draws (iteration 3)
    tho, lwo, ito, reco, d = oracle.smc_step(layers, a, X.astype(np.float64), y, win, mode, beta, sigma, kernel, seed,
                                             fraction, rkind, always, th0, lw0, 3)
    return rec, dump, th1, lw1, it1, reco, d, tho, lwo, ito


@pytest.mark.parametrize("S", [1, 3])
def test_smc_step_matches_oracle(product, oracle, S):
    rec, dump, th1, lw1, it1, reco, d, tho, lwo, ito = _step_compare(
        product, oracle, [64, 32, 10], "tanh", 2000, (0, 200, 2000), 0, 1.0, (0.002, S, 0), 32, 11, 0.5, 0, False)
    assert it1 == ito == 4
    assert rel(dump["log_target_old"], d["lt_old"]) < VAL_TOL
    assert rel(dump["log_target_new"], d["lt_new"]) < VAL_TOL
    # p_S - p0 = (h/2) (g_0 + 2 g_1 + ... + g_S): the gradient content of the final momentum.
    # Recovering it from fp32 momenta costs ulp(p)/(h/2) ~ 2.4e-4 absolute, i.e. ~3e-4 of the
    # max_rel_error floor here -- the bound is the fp32 storage of p, not the gradient
    # (the gradient itself is held to 1e-4 by test_value_and_grad_*).
    hh = 0.5 * 0.002
    for j in range(32):
        gsum, gsum_o = (dump["p_final"][j] - dump["p0"][j]) / hh, (d["pS"][j] - d["p0"][j]) / hh
        assert grad_err(gsum, gsum_o) < 3e-4
        nrm = np.linalg.norm(dump["p_final"][j] - d["pS"][j]) / np.linalg.norm(d["pS"][j])
        assert nrm < 2e-5, (j, nrm, np.abs(dump["p_final"][j] - d["pS"][j]).max(), np.abs(d["pS"][j]).max())
    np.testing.assert_allclose(rec["ess"], reco["ess"], rtol=1e-3)
    assert rec["resampled"] == reco["resampled"]
    if not rec["resampled"]:
        assert rel(lw1, lwo) < 1e-5
        for j in range(32):
            assert grad_err(th1[j], tho[j]) < GRAD_TOL


def test_smc_step_resample_always_systematic(product, oracle):
    rec, dump, th1, lw1, it1, reco, d, tho, lwo, ito = _step_compare(
        product, oracle, [12, 10, 4], "relu", 300, (0, 150, 300), 0, 1.0, (0.01, 2, 0), 64, 3, 1.0, 1, True)
    assert rec["resampled"] and reco["resampled"]
    assert np.max(np.abs(dump["weights"] - d["weights"])) < 1e-4
    # identical indices unless a uniform falls between the fp32/fp64 CDFs
    assert np.mean(dump["indices"] == d["indices"]) > 0.95
    np.testing.assert_allclose(lw1, lwo, rtol=1e-12)


def test_smc_step_sda_langevin(product, oracle):
    rec, dump, th1, lw1, it1, reco, d, tho, lwo, ito = _step_compare(
        product, oracle, [12, 10, 4], "tanh", 300, (100, 200, 300), 1, 0.3, (0.01, 1, 1), 16, 5, 0.5, 0, False)
    assert rel(dump["log_target_new"], d["lt_new"]) < VAL_TOL
    np.testing.assert_allclose(rec["ess"], reco["ess"], rtol=1e-3)


def test_divergence_and_all_dead(product, oracle):
    spec, X, y = make_problem(product, [6, 5, 3], "relu", 40)
    t = product.GpuEnsembleTarget(spec, X, y, 8)
    t.set_target(0, 40, 40, "scaled", 1.0, 1.0)
    t.init_ensemble(8, 1)
    with pytest.raises(product.SamplerError):
        t.smc_step(product.KernelConfig.hmc(1e30, 3), 1)


def test_determinism_and_c1_run(product, oracle):
    """Whole-run hot loop on C1 (BASELINE configs[0], shortened): schedule bit-exact,
    records reproducible on the GPU and close to the oracle."""
    layers = [64, 32, 10]
    spec, X, y = make_problem(product, layers, "tanh", 2000, seed=0, kind=0)
    cfg = product.RunConfig(kernel=product.KernelConfig.hmc(0.002, 3),
                            schedule=product.ScheduleConfig("ctr", 200, 100, 12, 2000, 1, 8),
                            particles=128, iterations=12, seed=0, resample="systematic")
    a = product.run_experiment(spec, X, y, cfg)["records"]
    b = product.run_experiment(spec, X, y, cfg)["records"]
    for ra, rb in zip(a, b):
        assert ra["ess"] == rb["ess"] and ra["mean_log_target"] == rb["mean_log_target"]
    o = oracle.run(layers, 1, X.astype(np.float64), y, kernel=(0.002, 3, 0), sched=(2, 200, 100, 1, 8),
                   particles=128, iterations=12, seed=0, resample_kind=1)
    assert [r["batch"] for r in a] == [r["batch"] for r in o] == [200] * 8 + [2000] * 4
    for ra, ro in zip(a[:3], o[:3]):
        np.testing.assert_allclose(ra["ess"], ro["ess"], rtol=1e-3)
        np.testing.assert_allclose(ra["mean_log_target"], ro["mean_log_target"], rtol=1e-5)


def test_sda_moments_and_run(product, oracle):
    layers = [8, 6, 2]
    spec, X, y = make_problem(product, layers, "relu", 400)
    t = product.GpuEnsembleTarget(spec, X, y, 32)
    t.set_target(0, 100, 400, "sda", 0.1, 1.0)
    t.init_ensemble(32, 4)
    th, lw, _ = t.get_ensemble(32)
    m = t.sda_moments(50, 150)
    a, b = oracle.loglik_parts(layers, 0, X.astype(np.float64), y, 50, 150, th)
    mo = oracle.sda_moments_from(-a, -b, lw)
    np.testing.assert_allclose(m, mo, rtol=1e-5, atol=1e-6 * np.max(np.abs(mo)))
    cfg = product.RunConfig(kernel=product.KernelConfig.hmc(0.01, 2),
                            schedule=product.ScheduleConfig("sda", 100, 100, 15, 400), particles=32, iterations=15,
                            seed=2)
    out = product.run_experiment(spec, X, y, cfg)
    betas = [s[0] for s in out["sda"]]
    assert all(0 < b_ <= 1 for b_ in betas)
    pre = [s[1] for s in out["sda"]]
    assert all(p2 >= p1 for p1, p2 in zip(pre, pre[1:]))


def test_constant_redraw_run(product, oracle):
    """Constant schedule with a fresh batch per iteration (runner.hpp:531-556): the device
    gathers train[draw_batch_rows(k)] and the window is {0, C, N}; records follow the oracle."""
    layers = [12, 10, 4]
    spec, X, y = make_problem(product, layers, "relu", 600)
    for prec in ("fp32", "tf32"):
        cfg = product.RunConfig(kernel=product.KernelConfig.hmc(0.01, 2),
                                schedule=product.ScheduleConfig("constant", 100, 100, 6, 600), particles=32,
                                iterations=6, seed=3, resample="systematic", redraw=True)
        a = product.run_experiment(spec, X, y, cfg, precision=prec if layers[0] % 4 == 0 else "fp32")["records"]
        o = oracle.run(layers, 0, X.astype(np.float64), y, kernel=(0.01, 2, 0), sched=(0, 100, 100, 1, -1),
                       redraw=True, particles=32, iterations=6, seed=3, resample_kind=1)
        assert [r["batch"] for r in a] == [r["batch"] for r in o] == [100] * 6
        for ra, ro in zip(a[:3], o[:3]):
            np.testing.assert_allclose(ra["ess"], ro["ess"], rtol=2e-3 if prec == "tf32" else 1e-3)
            np.testing.assert_allclose(ra["mean_log_target"], ro["mean_log_target"], rtol=1e-3 if prec == "tf32" else 1e-5)


@pytest.mark.parametrize("prec", ["fp32", "tf32"])
def test_sda_moments_fused_into_step(product, oracle, prec, monkeypatch):
    """after an SDA step the moments come from the step's own evaluations
    (kept positions for divergent particles, gathered through the resample) -- identical to
    the explicit forward pass on the post-step ensemble, and to the oracle within 1e-5."""
    layers = [12, 10, 4]
    spec, X, y = make_problem(product, layers, "relu", 400)
    res = {}
    for force in ("0", "1"):
        monkeypatch.setenv("DASMC_SDA_MOMENT_PASS", force)
        t = product.GpuEnsembleTarget(spec, X, y, 32, precision=prec if prec == "fp32" else "tf32")
        t.set_target(100, 250, 400, "sda", 0.3, 1.0)
        t.init_ensemble(32, 4)
        t.smc_step(product.KernelConfig.hmc(0.01, 2), 4, "multinomial", 1.0, True)
        res[force] = t.sda_moments(100, 250)
        th, lw, _ = t.get_ensemble(32)
        t.close()
    assert np.array_equal(res["0"], res["1"])
    a, b = oracle.loglik_parts(layers, 0, X.astype(np.float64), y, 100, 250, th)
    mo = oracle.sda_moments_from(-a, -b, lw)
    np.testing.assert_allclose(res["0"], mo, rtol=1e-5 if prec == "fp32" else 1e-3,
                               atol=(1e-6 if prec == "fp32" else 1e-3) * np.max(np.abs(mo)))


@pytest.mark.parametrize("prec", ["fp32", "tf32"])
def test_start_gradient_cache_is_exact(product, prec):
    """SURVEY.md §8f.1 / SPEC.md:410: with an unchanged target the cached start log targets and
    gradients equal the recomputed ones, so the chain is bit-identical with S instead of S+1
    evaluations per step; a target change falls back to recomputing."""
    layers = [16, 12, 4]
    spec, X, y = make_problem(product, layers, "tanh", 300)
    runs = {}
    for cache in (False, True):
        t = product.GpuEnsembleTarget(spec, X, y, 24, precision=prec)
        t.set_target(0, 200, 300, "scaled", 1.0, 1.0)
        t.init_ensemble(24, 9)
        if cache:
            t.set_cache_start(True)
        recs, used = [], []
        for k in range(5):
            if k == 3:
                t.set_target(0, 250, 300, "scaled", 1.0, 1.0)  # window grows: no cache this step
            recs.append(t.smc_step(product.KernelConfig.hmc(0.01, 3), 9, "systematic", 0.5))
            used.append(t.last_step_cached())
        th, lw, _ = t.get_ensemble(24)
        runs[cache] = (th, lw, recs, used)
        t.close()
    assert runs[True][3] == [False, True, True, False, True]
    assert np.array_equal(runs[False][0], runs[True][0]) and np.array_equal(runs[False][1], runs[True][1])
    for a, b in zip(runs[False][2], runs[True][2]):
        assert a["ess"] == b["ess"] and a["mean_log_target"] == b["mean_log_target"]


def test_bench_memory_hook(product):
    """dasmc_gpu_bench_memory (tools/membench.py): runs every memory-bound kernel of the
    step on the context's buffers and reports positive times and the algorithmic bytes."""
    import ctypes as C
    from paper_2601_21983_b200 import _lib as L
    spec, X, y = make_problem(product, [30, 20, 5], "relu", 64)
    J = 300
    t = product.GpuEnsembleTarget(spec, X, y, J)
    t.init_ensemble(J, 1)
    idx = np.random.default_rng(0).integers(0, J, J).astype(np.int32)
    ms, by = np.zeros(4), np.zeros(4)
    L.check(t.lib.dasmc_gpu_bench_memory(t.h, J, idx.ctypes.data_as(C.POINTER(C.c_int32)), 2,
                                         ms.ctypes.data_as(C.POINTER(C.c_double)),
                                         by.ctypes.data_as(C.POINTER(C.c_double))))
    assert np.all(ms > 0) and np.all(np.isfinite(ms)), ms
    D = product.param_count(spec)
    assert by[2] == 4.0 * J * D and by[0] >= 8.0 * J * D
    bad = idx.copy()
    bad[0] = J
    with pytest.raises(ValueError):
        L.check(t.lib.dasmc_gpu_bench_memory(t.h, J, bad.ctypes.data_as(C.POINTER(C.c_int32)), 1,
                                             ms.ctypes.data_as(C.POINTER(C.c_double)),
                                             by.ctypes.data_as(C.POINTER(C.c_double))))
    t.close()


def test_particle_count_bounds(product):
    """max_particles is bounded per context (2 .. 65535: the gather kernels index particles by gridDim.y,
    ADVICE r1); out-of-range values are invalid arguments, not launch failures."""
    spec, X, y = make_problem(product, [6, 4, 3], "tanh", 16)
    for bad in (1, 65536, 100000):
        with pytest.raises(ValueError):
            product.GpuEnsembleTarget(spec, X, y, bad)

"""GPU parity of the tensor-core CNN stages (conv_tc.cu: tcgen05 kind::tf32 implicit GEMMs) and
of the chunked CNN window (memory independent of M) against the fp64 oracle.

The reference is MLP-only (network.hpp:21-27); its contraction sites network.hpp:171-173
(forward) and 203-209 (weight gradient, delta) are generalised to convolution stages
(BASELINE.json configs[2..3]); the oracle's CnnSpec is pinned to torch fp64 autograd in
test_oracle_pins.py.

Stated tolerances of the tensor-core CNN path (tf32 operands rounded to nearest, fp32
accumulation; the MLP head stays fp32 on CUDA cores), measured on B200:
  values    relative 2e-4 of |log target|;
  gradients normwise ||g - ref|| / ||ref|| < 3e-2 per particle (measured: C3 5.8e-3, C4 1.5e-2;
  like the deep tf32 MLPs in test_gpu_tensorcore.py, the error grows with depth as the tf32
  forward moves a few ReLU pre-activations across zero against the fp64 oracle).
The fp32 CUDA-core path (precision="fp32") keeps the 1e-4 bounds of test_gpu_cnn.py,
chunked or not.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

C3 = (((1, 28, 28), [(5, 16, True), (5, 32, True)]), [512, 10], "relu")
C4 = (((3, 32, 32), [(3, 32, False), (3, 32, True), (3, 64, False), (3, 64, True)]), [1600, 256, 10], "relu")
# odd sizes (floor pooling), tanh, a last stage without a pool (NHWC <-> flatten permutes)
ODD = (((2, 11, 11), [(3, 4, True), (2, 8, False)]), [8 * 3 * 3, 6, 3], "tanh")
# wider input (slab lines padded from 18 / 16 to a pitch of 32 / 16), three stages, a pooled last stage
WIDE = (((3, 40, 40), [(5, 32, True), (3, 64, False), (3, 32, True)]), [32 * 7 * 7, 10], "relu")
# narrow channel counts: 8-channel pooled outputs padded to a 32-channel block (one data-carrying k-step),
# k = 2 kernels, a 12-channel stage (not a multiple of 8: the gather-form weight gradient with kx-shifted
# copies and the staged pool backward), tanh
NARROW = (((1, 20, 20), [(3, 8, True), (2, 16, True), (3, 12, False)]), [12 * 2 * 2, 5], "tanh")
VAL_TC, GRAD_TC = 2e-4, 3e-2


def rel(a, b):
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300)))


def norm_err(g, ref):
    return float(np.linalg.norm(g - ref) / np.linalg.norm(ref))


def max_rel_error(a, b, floor):  # test_util.hpp:37-45
    return float(np.max(np.abs(a - b) / np.maximum(np.maximum(np.abs(a), np.abs(b)), floor)))


def problem(product, arch, n, kind=1):
    conv, head, act = arch
    spec = product.NetSpec(head, act, conv)
    X, y = product.make_teacher_data(spec, n, kind, 0, 3, threads=8)
    return spec, X, y


@pytest.mark.parametrize("arch,M,J", [(C3, 40, 3), (C4, 12, 2), (ODD, 50, 4), (WIDE, 10, 2), (NARROW, 40, 3)])
def test_cnn_tc_value_and_grad(product, oracle, arch, M, J):
    n = 64
    spec, X, y = problem(product, arch, n)
    D = product.param_count(spec)
    th = (0.3 * np.random.default_rng(1).standard_normal((J, D))).astype(np.float32).astype(np.float64)
    t = product.GpuEnsembleTarget(spec, X, y, J, precision="tf32")
    a = 0 if arch[2] == "relu" else 1
    for mode, win, beta, sigma in (("scaled", (0, M, n), 1.0, 1.0), ("sda", (M // 3, M, n), 0.4, 0.7)):
        t.set_target(*win, mode, beta, sigma)
        v, g = t.log_target_with_grad(th)
        vo, go = oracle.value_and_grad(spec.oracle_layers(), a, X.astype(np.float64), y, win,
                                       0 if mode == "scaled" else 1, beta, sigma, th)
        errs = [norm_err(g[j], go[j]) for j in range(J)]
        print(f"tc cnn {arch[1]} M={M} {mode}: value rel {rel(v, vo):.2e} grad norm {max(errs):.2e}")
        assert rel(v, vo) < VAL_TC, (mode, v, vo)
        assert max(errs) < GRAD_TC, (mode, errs)
    t.close()


@pytest.mark.parametrize("prec", ["fp32", "tf32"])
def test_cnn_chunked_window(product, oracle, prec, monkeypatch):
    """A window of 300 images evaluated in chunks of 128 (gradient sums carried across chunks
    before the fused leapfrog) matches the oracle and the single-chunk evaluation."""
    spec, X, y = problem(product, ODD, 320)
    D = product.param_count(spec)
    J = 3
    th = (0.3 * np.random.default_rng(2).standard_normal((J, D))).astype(np.float32).astype(np.float64)
    win = (100, 300, 320)
    vo, go = oracle.value_and_grad(spec.oracle_layers(), 1, X.astype(np.float64), y, win, 1, 0.6, 1.0, th)
    out = {}
    for chunk in (None, "128"):
        if chunk:
            monkeypatch.setenv("DASMC_CNN_CHUNK", chunk)
        else:
            monkeypatch.delenv("DASMC_CNN_CHUNK", raising=False)
        t = product.GpuEnsembleTarget(spec, X, y, J, precision=prec)
        t.set_target(*win, "sda", 0.6, 1.0)
        out[chunk] = t.log_target_with_grad(th)
        t.close()
    for v, g in out.values():
        if prec == "fp32":
            assert rel(v, vo) < 1e-5
            for j in range(J):
                assert max_rel_error(g[j], go[j], 1e-3 * np.max(np.abs(go[j]))) < 1e-4
        else:
            assert rel(v, vo) < VAL_TC
            assert max(norm_err(g[j], go[j]) for j in range(J)) < GRAD_TC
    (v1, g1), (v2, g2) = out[None], out["128"]
    # fp32 reassociation of the window sums: CUDA-core path 1e-5, tensor-core accumulation 1e-4
    assert rel(v2, v1) < 1e-6 and max(norm_err(g2[j], g1[j]) for j in range(J)) < (1e-5 if prec == "fp32" else 1e-4)


def test_cnn_smc_step_tc(product, oracle):
    spec, X, y = problem(product, ODD, 120)
    lay = spec.oracle_layers()
    J, seed = 16, 5
    win = (0, 90, 120)
    th0, lw0 = oracle.init_ensemble(lay, 1, X.astype(np.float64), y, win, 0, 1.0, 1.0, seed, J)
    th0 = th0.astype(np.float32).astype(np.float64)
    t = product.GpuEnsembleTarget(spec, X, y, J, precision="tf32")
    t.set_target(*win, "scaled", 1.0, 1.0)
    t.set_ensemble(th0, lw0, 3)
    rec = t.smc_step(product.KernelConfig.hmc(0.005, 2), seed, "multinomial", 0.5)
    dump = t.last_proposals(J)
    t.close()
    _, _, _, reco, d = oracle.smc_step(lay, 1, X.astype(np.float64), y, win, 0, 1.0, 1.0, (0.005, 2, 0), seed, 0.5, 0,
                                       False, th0, lw0, 3)
    assert rel(dump["log_target_old"], d["lt_old"]) < VAL_TC
    assert rel(dump["log_target_new"], d["lt_new"]) < VAL_TC
    np.testing.assert_allclose(rec["ess"], reco["ess"], rtol=2e-2)


@pytest.mark.parametrize("prec", ["fp32", "tf32"])
def test_c3_many_particles_long_window(product, oracle, prec):
    """J = 512 particles at M = 2100 images (J * ceil(M / 16) > 65535 conv
    weight-gradient blocks before the window was chunked).  Particle j's result must not depend
    on J: compare with a 2-particle context (values bit-identical; gradients to fp32
    reassociation: the two contexts split the window into different chunks, and the tensor
    cores' fp32 accumulation over K = 2100 x 64 pixels differs at ~1e-3), and the first
    particle's value and gradient with the oracle."""
    spec, X, y = problem(product, C3, 2100)
    D = product.param_count(spec)
    J = 512
    th = (0.2 * np.random.default_rng(4).standard_normal((J, D))).astype(np.float32).astype(np.float64)
    t = product.GpuEnsembleTarget(spec, X, y, J, precision=prec)
    t.set_target(0, 2100, 2100, "scaled", 1.0, 1.0)
    v, g = t.log_target_with_grad(th)
    t.close()
    t1 = product.GpuEnsembleTarget(spec, X, y, 2, precision=prec)
    t1.set_target(0, 2100, 2100, "scaled", 1.0, 1.0)
    v1, g1 = t1.log_target_with_grad(th[[0, J - 1]])
    t1.close()
    assert np.all(np.isfinite(v)) and np.all(np.isfinite(g))
    np.testing.assert_array_equal(v[[0, J - 1]], v1)
    for a, b in zip(g[[0, J - 1]], g1):
        assert norm_err(a, b) < (1e-6 if prec == "fp32" else 3e-3)
    vo, go = oracle.value_and_grad(spec.oracle_layers(), 0, X.astype(np.float64), y, (0, 2100, 2100), 0, 1.0, 1.0,
                                   th[:1])
    print(f"{prec} M=2100 J=512: value rel {rel(v[:1], vo):.2e} grad norm {norm_err(g[0], go[0]):.2e} "
          f"(J=2 context: {norm_err(g1[0], go[0]):.2e})")
    assert rel(v[:1], vo) < (1e-5 if prec == "fp32" else VAL_TC)
    tol = 1e-4 if prec == "fp32" else GRAD_TC
    assert norm_err(g[0], go[0]) < tol and norm_err(g1[0], go[0]) < tol


@pytest.mark.parametrize("arch,J", [(C3, 251), (C4, 189)])
def test_stage0_particle_batching_tail(product, oracle, arch, J, monkeypatch):
    """The stage-0 GEMMs put several particles on the MMA's N dimension (the im2col of X and its transpose
    are shared by every particle).  J is not a multiple of the batch, so the last unit's missing particles
    are zero rows; the weight-gradient batch is forced to 4 (the heuristic keeps one particle per unit at
    this small J).  Particles at the start, across a batch boundary and in the tail match the oracle, and
    equal the unbatched evaluation (values bit-identical, gradients to fp32 reassociation)."""
    M, n = 24, 32
    spec, X, y = problem(product, arch, n)
    D = product.param_count(spec)
    th = (0.2 * np.random.default_rng(8).standard_normal((J, D))).astype(np.float32).astype(np.float64)
    monkeypatch.setenv("DASMC_CONV_NBW", "4")
    t = product.GpuEnsembleTarget(spec, X, y, J, precision="tf32")
    t.set_target(0, M, n, "scaled", 1.0, 1.0)
    v, g = t.log_target_with_grad(th)
    t.close()
    monkeypatch.delenv("DASMC_CONV_NBW")
    monkeypatch.setenv("DASMC_CONV_BATCH0", "0")
    t = product.GpuEnsembleTarget(spec, X, y, J, precision="tf32")
    t.set_target(0, M, n, "scaled", 1.0, 1.0)
    v0, g0 = t.log_target_with_grad(th)
    t.close()
    assert np.all(np.isfinite(v)) and np.all(np.isfinite(g))
    np.testing.assert_array_equal(v, v0)
    assert max(norm_err(g[j], g0[j]) for j in range(J)) < 1e-5
    pick = [0, 3, 4, 15, 16, J - 2, J - 1]
    vo, go = oracle.value_and_grad(spec.oracle_layers(), 0, X.astype(np.float64), y, (0, M, n), 0, 1.0, 1.0, th[pick])
    assert rel(v[pick], vo) < VAL_TC
    assert max(norm_err(g[j], go[i]) for i, j in enumerate(pick)) < GRAD_TC


@pytest.mark.parametrize("arch", [C3, C4])
@pytest.mark.parametrize("switch", ["DASMC_CONV_FOLD", "DASMC_CONV_PERSIST", "DASMC_CONV_CPAD", "DASMC_CONV_DWT",
                                    "DASMC_CONV_DIRECT"])
def test_conv_path_switches_agree(product, oracle, arch, switch, monkeypatch):
    """The tensor-core stages choose among operand-feed forms (conv_tc.cu: kx fold + padded slab lines,
    resident weights, channel-padded pooled outputs, TMA weight gradients with shared-memory shifts, direct
    convolutions vs gathers).  Each form switched off must give the same log target (bit-identical: the
    forward operands and accumulation order per pixel do not change... except where the fold reassociates the
    sum over kx, so values are compared to 1e-6 relative) and the same gradient to fp32 reassociation, and
    both must meet the oracle bound."""
    M, n, J = 24, 32, 3
    spec, X, y = problem(product, arch, n)
    D = product.param_count(spec)
    th = (0.2 * np.random.default_rng(9).standard_normal((J, D))).astype(np.float32).astype(np.float64)

    def run():
        t = product.GpuEnsembleTarget(spec, X, y, J, precision="tf32")
        t.set_target(0, M, n, "scaled", 1.0, 1.0)
        out = t.log_target_with_grad(th)
        t.close()
        return out

    v, g = run()
    monkeypatch.setenv(switch, "0")
    v0, g0 = run()
    assert rel(v, v0) < 1e-6
    assert max(norm_err(g[j], g0[j]) for j in range(J)) < 2e-3
    vo, go = oracle.value_and_grad(spec.oracle_layers(), 0, X.astype(np.float64), y, (0, M, n), 0, 1.0, 1.0, th)
    for vv, gg in ((v, g), (v0, g0)):
        assert rel(vv, vo) < VAL_TC
        assert max(norm_err(gg[j], go[j]) for j in range(J)) < GRAD_TC


def test_c4_full_batch_window(product):
    """BASELINE configs[3]'s full-batch phase: a window of all n = 50000 images (tensor-core
    stages, chunked).  Size-independent checks: finite values and gradients, and additivity of
    the unscaled log-likelihood: prefix [0, P) + block [P, M) equals the scaled target's data
    term (target.hpp:121-173)."""
    spec, X, y = problem(product, C4, 50000)
    D = product.param_count(spec)
    J = 4
    th = (0.05 * np.random.default_rng(6).standard_normal((J, D))).astype(np.float32).astype(np.float64)
    t = product.GpuEnsembleTarget(spec, X, y, J, precision="tf32")
    t.set_target(0, 50000, 50000, "scaled", 1.0, 1.0)
    v, g = t.log_target_with_grad(th)
    assert np.all(np.isfinite(v)) and np.all(np.isfinite(g))
    t.set_target(20000, 50000, 50000, "sda", 1.0, 1.0)
    a, b = t.unscaled_loglik_parts(th)
    t.close()
    prior = -0.5 * D * np.log(2 * np.pi) - 0.5 * np.sum(th * th, axis=1)
    np.testing.assert_allclose(prior + a + b, v, rtol=1e-6)

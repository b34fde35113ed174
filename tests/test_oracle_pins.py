"""CPU: pin the oracle -- the reference's own known answers (ported Catch2
tests, oracle/oracle_tests.cpp) and the committed golden vectors."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden", "golden.npz")


def test_reference_kats_ported(oracle):
    if not os.path.exists(oracle.TESTS_BIN):
        oracle.build()
    r = subprocess.run([oracle.TESTS_BIN], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout


@pytest.fixture(scope="module")
def gold():
    return dict(np.load(GOLD))


def test_golden_rng(oracle, gold):
    keys = [oracle.fork_key(s, a, b, c) for s in (0, 1, 42) for a in (1, 2, 3) for b in (0, 7) for c in (0, 5)]
    assert np.array_equal(np.array(keys, dtype=np.uint64), gold["fork_keys"])
    assert np.array_equal(oracle.rng_u64(oracle.fork_key(0, 2, 0, 0), 64), gold["u64"])
    assert np.array_equal(oracle.rng_normals(oracle.fork_key(3, 2, 1, 4), 256), gold["normals"])
    assert np.array_equal(oracle.rng_uniforms(oracle.fork_key(3, 3, 9, 0), 256), gold["uniforms"])


def test_golden_data(oracle, gold):
    X, y = oracle.make_teacher([8, 4, 3], 0, 50, 0, 11, 1)
    assert np.array_equal(X, gold["teacher_X"]) and np.array_equal(y, gold["teacher_y"])
    assert np.array_equal(oracle.shuffle_perm(0, 100), gold["perm"])


def test_golden_value_and_grad(oracle, gold):
    layers = [64, 32, 10]
    Xc, yc = oracle.make_teacher(layers, 1, 300, 0, 0, 1)
    v, g = oracle.value_and_grad(layers, 1, Xc, yc, (0, 100, 300), 0, 1.0, 1.0, gold["vg_theta"])
    np.testing.assert_allclose(v, gold["vg_scaled_values"], rtol=1e-12)
    np.testing.assert_allclose(g, gold["vg_scaled_grads"], rtol=1e-10, atol=1e-10)


def test_golden_smc_step(oracle, gold):
    layers2 = [6, 5, 3]
    X2, y2 = oracle.make_teacher(layers2, 0, 40, 0, 3, 1)
    th0, lw0 = oracle.init_ensemble(layers2, 0, X2, y2, (0, 20, 40), 0, 1.0, 1.0, 5, 8)
    np.testing.assert_array_equal(th0, gold["init_theta"])
    th1, lw1, _, rec, d = oracle.smc_step(layers2, 0, X2, y2, (0, 20, 40), 0, 1.0, 1.0, (0.05, 3, 0), 5, 1.0, 0,
                                          False, th0, lw0, 0)
    np.testing.assert_allclose(th1, gold["step_theta"], rtol=1e-12, atol=1e-12)
    np.testing.assert_array_equal(d["indices"], gold["step_indices"])


def test_golden_schedules(oracle, gold):
    for i, kind in enumerate((0, 1, 2, 3, 4)):
        got = [oracle.batch_size(kind, 500, 500, 200, 60000, 1, -1, k) for k in range(200)]
        assert got == list(gold["schedules"][i])
    # SPEC.md annealing KATs inside the frozen table
    assert gold["schedules"][2][179] == 500 and gold["schedules"][2][180] == 60000
    assert gold["schedules"][4][1] == 1000


# ---- [EXT] CNN layers: no reference oracle exists (the reference is MLP-only), so the
# oracle's conv / pool / flatten restatement is pinned to torch fp64 autograd and to
# central finite differences.
def _torch_cnn_ll(spec, th, X, y):
    torch = pytest.importorskip("torch")
    (c, h, w), convs, head, act = spec
    f = torch.relu if act == 0 else torch.tanh
    x = torch.tensor(X, dtype=torch.float64).reshape(-1, c, h, w)
    t = torch.tensor(th, dtype=torch.float64, requires_grad=True)
    off, cin = 0, c
    for k, co, pool in convs:
        W = t[off:off + co * cin * k * k].reshape(co, cin, k, k)
        off += co * cin * k * k
        b = t[off:off + co]
        off += co
        x = f(torch.nn.functional.conv2d(x, W, b))
        if pool:
            x = torch.nn.functional.max_pool2d(x, 2)
        cin = co
    a = x.reshape(x.shape[0], -1)
    for l in range(1, len(head)):
        i, o = head[l - 1], head[l]
        W = t[off:off + i * o].reshape(i, o)  # reference W (out x in) column-major == row-major [in][out]
        off += i * o
        b = t[off:off + o]
        off += o
        a = a @ W + b
        if l + 1 < len(head):
            a = f(a)
    ll = torch.log_softmax(a, 1)[torch.arange(len(y)), torch.tensor(y, dtype=torch.long)].sum()
    ll.backward()
    return float(ll), t.grad.numpy()


@pytest.mark.parametrize("spec", [((1, 14, 14), [(5, 4, True), (3, 6, True)], [6 * 1 * 1, 10], 0),
                                  ((3, 10, 10), [(3, 4, False), (3, 5, True)], [5 * 3 * 3, 7, 4], 1),
                                  ((2, 9, 9), [(2, 3, True)], [3 * 4 * 4, 5], 0)])
def test_cnn_oracle_matches_torch_autograd(oracle, spec):
    (c, h, w), convs, head, act = spec
    lay = oracle.cnn_layers((c, h, w), convs, head)
    D = oracle.param_count(lay)
    X, y = oracle.make_teacher(lay, act, 30, 1, 0, 4, 1)
    th = 0.4 * np.random.default_rng(2).standard_normal((2, D))
    v, g = oracle.value_and_grad(lay, act, X, y, (0, 30, 30), 0, 1.0, 1.0, th)
    for j in range(2):
        ll, gt = _torch_cnn_ll(spec, th[j], X, y)
        prior = -0.5 * D * np.log(2 * np.pi) - 0.5 * np.sum(th[j] ** 2)
        assert abs(v[j] - (ll + prior)) < 1e-10 * abs(v[j])
        np.testing.assert_allclose(g[j], gt - th[j], rtol=1e-9, atol=1e-11)


def test_cnn_oracle_finite_differences(oracle):
    lay = oracle.cnn_layers((1, 8, 8), [(3, 2, True), (2, 3, False)], [3 * 2 * 2, 4])
    D = oracle.param_count(lay)
    X, y = oracle.make_teacher(lay, 1, 12, 0, 0, 5, 1)
    th = 0.5 * np.random.default_rng(6).standard_normal((1, D))
    _, g = oracle.value_and_grad(lay, 1, X, y, (0, 12, 12), 0, 1.0, 1.0, th)
    eps = 1e-6
    for i in np.random.default_rng(7).choice(D, 25, replace=False):
        tp, tm = th.copy(), th.copy()
        tp[0, i] += eps
        tm[0, i] -= eps
        vp, _ = oracle.value_and_grad(lay, 1, X, y, (0, 12, 12), 0, 1.0, 1.0, tp, want_grad=False)
        vm, _ = oracle.value_and_grad(lay, 1, X, y, (0, 12, 12), 0, 1.0, 1.0, tm, want_grad=False)
        assert abs((vp[0] - vm[0]) / (2 * eps) - g[0, i]) < 1e-5 * max(1.0, abs(g[0, i]))

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

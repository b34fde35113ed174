"""GPU evaluate_predictive (runner.hpp:331-364) against the oracle."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("prec", ["fp32", "tf32"])
def test_evaluate_predictive_mlp(product, oracle, prec):
    layers = [784, 200, 10]
    spec = product.NetSpec(layers, "relu")
    X, y = product.make_teacher_data(spec, 3000, 1, 0, 2, threads=8)
    Xtr, ytr, Xte, yte = X[:2000], y[:2000], X[2000:], y[2000:]
    J = 24
    th, lw = oracle.init_ensemble(layers, 0, Xtr.astype(np.float64), ytr, (0, 500, 2000), 0, 1.0, 1.0, 3, J)
    th = th.astype(np.float32).astype(np.float64)
    lw[3] = -np.inf  # a dead particle contributes nothing
    t = product.GpuEnsembleTarget(spec, Xtr, ytr, J, precision=prec)
    t.set_target(0, 500, 2000, "scaled", 1.0, 1.0)
    t.set_ensemble(th, lw, 0)
    lp, acc = t.evaluate_predictive(Xte, yte)
    lpo, acco = oracle.evaluate_predictive(layers, 0, Xte.astype(np.float64), yte, th, lw)
    assert abs(lp - lpo) < 1e-5 * abs(lpo)
    assert abs(acc - acco) <= 100.0 / len(yte) + 1e-9  # at most one near-tie row may flip
    # sharded form: two halves mixed and summed equal the whole
    w = np.exp(lw - lw.max())
    w /= w.sum()
    pred = np.zeros((len(yte), 10))
    t.predictive_mix(Xte, w, J, pred)
    assert np.allclose(product.predictive_metrics(pred, yte), (lp, acc), rtol=1e-12)


def test_evaluate_predictive_cnn(product, oracle):
    conv = ((1, 12, 12), [(3, 4, True), (3, 6, False)])
    spec = product.NetSpec([54, 7, 5], "relu", conv)
    lay = spec.oracle_layers()
    X, y = product.make_teacher_data(spec, 400, 1, 0, 3, threads=8)
    J = 6
    th, lw = oracle.init_ensemble(lay, 0, X[:300].astype(np.float64), y[:300], (0, 100, 300), 0, 1.0, 1.0, 4, J)
    th = th.astype(np.float32).astype(np.float64)
    t = product.GpuEnsembleTarget(spec, X[:300], y[:300], J)
    t.set_target(0, 100, 300, "scaled", 1.0, 1.0)
    t.set_ensemble(th, lw, 0)
    lp, acc = t.evaluate_predictive(X[300:], y[300:])
    lpo, acco = oracle.evaluate_predictive(lay, 0, X[300:].astype(np.float64), y[300:], th, lw)
    assert abs(lp - lpo) < 1e-5 * abs(lpo)
    assert abs(acc - acco) <= 100.0 / 100 + 1e-9

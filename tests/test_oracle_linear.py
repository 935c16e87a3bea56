"""Linear-model oracle (oracle.c oracle_linear_run) pinned to
hand-computed values (tests/golden/linear_models_hand.json) and to
scikit-learn's own routines: LogisticRegression (binary / multinomial),
LinearRegression, Ridge, SGDClassifier, and StandardScaler.transform (bitwise,
reading c16) through an identity model."""
from types import SimpleNamespace

import numpy as np
import pytest

import oracle
from synth import gen_x
from tests.helpers import load_golden, parse_x


def _lin(coef, intercept=None, mean=None, scale=None, task=1, post=0):
    coef = np.asarray(coef, np.float64)
    return SimpleNamespace(n_features=coef.shape[1], n_outputs=coef.shape[0], coef=coef,
                           intercept=None if intercept is None else np.asarray(intercept, np.float64),
                           mean=None if mean is None else np.asarray(mean, np.float64),
                           scale=None if scale is None else np.asarray(scale, np.float64), task=task, post=post)


@pytest.mark.parametrize("case", ["binary", "binary_scaled", "multiclass"])
def test_linear_hand_golden(case):
    g = load_golden("linear_models_hand.json")
    c = g[case]
    m = _lin(c["coef"], c["intercept"], c.get("mean"), c.get("scale"), task=1, post=2 if case == "multiclass" else 1)
    o = oracle.run_linear(m, parse_x(g["X"]))
    np.testing.assert_array_equal(o["s"].reshape(np.asarray(c["s"]).shape if case == "multiclass" else -1),
                                  np.asarray(c["s"]))
    assert o["label"].tolist() == c["label"]
    if case == "multiclass":
        np.testing.assert_allclose(o["proba"], np.asarray(c["proba"]), rtol=1e-6)
    else:
        np.testing.assert_allclose(o["proba"][:, 1], c["p1"], rtol=1e-6)


sk = pytest.importorskip("sklearn")


def _data(seed, n, F, k):
    X = gen_x(seed, 0, n, F) * np.float32(3.0) + np.float32(1.0)
    z = X @ np.linspace(-1, 1, F).astype(np.float32)
    y = np.digitize(z, np.quantile(z, np.linspace(0, 1, k + 1)[1:-1]))
    return X, y, z


def _f64(X):
    # the same (fp32-representable) values in float64: sklearn then keeps fp64
    # coefficients and computes the library reference in fp64, like the oracle
    return X.astype(np.float64)


def test_standard_scaler_transform_bitwise():
    from sklearn.preprocessing import StandardScaler
    X, _, _ = _data(61, 2000, 7, 2)
    sc = StandardScaler().fit(X)
    Xt = gen_x(62, 0, 500, 7) * np.float32(3.0)
    m = _lin(np.eye(7), None, sc.mean_, sc.scale_, task=0)
    o = oracle.run_linear(m, Xt)
    np.testing.assert_array_equal(o["pred"], sc.transform(Xt))


@pytest.mark.parametrize("k,scaled", [(2, False), (4, False), (3, True)])
def test_logistic_regression(k, scaled):
    from sklearn.linear_model import LogisticRegression
    from sklearn.preprocessing import StandardScaler
    X, y, _ = _data(63, 3000, 9, k)
    sc = StandardScaler().fit(X) if scaled else None
    lr = LogisticRegression(max_iter=500).fit(_f64(sc.transform(X) if scaled else X), y)
    Xt, _, _ = _data(64, 2000, 9, k)
    K = lr.coef_.shape[0]
    m = _lin(lr.coef_, lr.intercept_, None if sc is None else sc.mean_, None if sc is None else sc.scale_,
             task=1, post=1 if K == 1 else 2)
    o = oracle.run_linear(m, Xt)
    Xs = _f64(sc.transform(Xt) if scaled else Xt)  # fp32 scaler output (c16), fp64 model
    d = lr.decision_function(Xs).reshape(len(Xt), -1)
    np.testing.assert_allclose(o["s"], d, rtol=1e-12, atol=1e-12)
    p = lr.predict_proba(Xs)
    np.testing.assert_allclose(o["proba"], p, rtol=1e-5, atol=1e-7)
    gap = np.abs(d[:, 0]) if K == 1 else -np.diff(np.sort(d, axis=1)[:, -2:], axis=1)[:, 0]
    clear = gap > 1e-9
    np.testing.assert_array_equal(o["label"][clear], lr.predict(Xs)[clear])


def test_linear_and_ridge_regression_multioutput():
    from sklearn.linear_model import LinearRegression, Ridge
    X, _, z = _data(65, 2000, 6, 2)
    Y = np.stack([z, 0.5 * z + X[:, 0]], 1)
    Xt, _, _ = _data(66, 1000, 6, 2)
    for est in (LinearRegression().fit(_f64(X), Y), Ridge(alpha=0.3).fit(_f64(X), Y)):
        m = _lin(est.coef_, est.intercept_, task=0)
        o = oracle.run_linear(m, Xt)
        np.testing.assert_allclose(o["s"], est.predict(_f64(Xt)), rtol=1e-12, atol=1e-9)


def test_sgd_classifier_hinge():
    from sklearn.linear_model import SGDClassifier
    X, y, _ = _data(67, 3000, 8, 3)
    est = SGDClassifier(random_state=0, max_iter=50, tol=None).fit(_f64(X), y)
    Xt, _, _ = _data(68, 1000, 8, 3)
    m = _lin(est.coef_, est.intercept_, task=1, post=0)
    o = oracle.run_linear(m, Xt)
    d = est.decision_function(_f64(Xt))
    np.testing.assert_allclose(o["s"], d, rtol=1e-12, atol=1e-9)
    clear = -np.diff(np.sort(d, axis=1)[:, -2:], axis=1)[:, 0] > 1e-9
    np.testing.assert_array_equal(o["label"][clear], est.predict(_f64(Xt))[clear])

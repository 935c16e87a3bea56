"""Oracle pinned to a library routine: scikit-learn's own tree apply/predict
(sklearn _tree.pyx _apply_dense: x <= threshold -> left, NaN -> missing_go_to_left;
_forest.py predict_proba: mean of per-tree fractions; _gb.py: init + lr * sum).
apply must be bit-exact; labels exact where sklearn's top-2 gap > 1e-4 (SPEC.md:333
gap guard); probabilities/scores within 1e-5 (fp32 leaf-value rounding, reading c5)."""
import numpy as np
import pytest

import oracle
from synth import gen_x, inject_specials
from tests.sk_export import from_sklearn_forest, from_sklearn_gbc_multiclass, from_sklearn_gbr

sk = pytest.importorskip("sklearn")
from sklearn.ensemble import GradientBoostingClassifier, GradientBoostingRegressor, RandomForestClassifier  # noqa: E402
from sklearn.tree import DecisionTreeClassifier  # noqa: E402


def _data(seed, n, F, n_classes, nan_rate=0.0):
    X = gen_x(seed, 0, n, F)
    w = np.linspace(-1, 1, F).astype(np.float32)
    z = X @ w + 0.3 * X[:, 0] * X[:, -1]
    y = np.digitize(z, np.quantile(z, np.linspace(0, 1, n_classes + 1)[1:-1]))
    if nan_rate:
        X = inject_specials(X, seed, rate=nan_rate)
        X[np.isinf(X)] = 0.0
    return X, y, z


def _check_labels(p_sk, lab_ours):
    srt = np.sort(p_sk, axis=1)
    clear = (srt[:, -1] - srt[:, -2]) > 1e-4
    assert clear.mean() > 0.5
    np.testing.assert_array_equal(np.argmax(p_sk, axis=1)[clear], lab_ours[clear])


@pytest.mark.parametrize("nan_rate", [0.0, 0.02])
def test_decision_tree_classifier(nan_rate):
    X, y, _ = _data(21, 3000, 6, 3, nan_rate)
    est = DecisionTreeClassifier(max_depth=7, random_state=0).fit(X, y)
    m = from_sklearn_forest(est, 6, with_missing=nan_rate > 0)
    Xt, _, _ = _data(22, 2000, 6, 3, nan_rate)
    o = oracle.run(m, Xt)
    np.testing.assert_array_equal(o["leaf"][:, 0], est.apply(Xt))
    p = est.predict_proba(Xt)
    np.testing.assert_allclose(o["proba"], p, atol=1e-6)
    _check_labels(p, o["label"])


@pytest.mark.parametrize("nan_rate", [0.0, 0.02])
def test_random_forest_classifier(nan_rate):
    X, y, _ = _data(31, 3000, 8, 4, nan_rate)
    est = RandomForestClassifier(n_estimators=25, max_depth=8, random_state=0).fit(X, y)
    m = from_sklearn_forest(est, 8, with_missing=nan_rate > 0)
    Xt, _, _ = _data(32, 2000, 8, 4, nan_rate)
    o = oracle.run(m, Xt)
    np.testing.assert_array_equal(o["leaf"], est.apply(Xt))
    p = est.predict_proba(Xt)
    np.testing.assert_allclose(o["proba"], p, atol=1e-6)
    _check_labels(p, o["label"])


def test_gradient_boosting_regressor():
    X, _, z = _data(41, 3000, 5, 2)
    est = GradientBoostingRegressor(n_estimators=40, max_depth=4, learning_rate=0.1,
                                    random_state=0).fit(X, z)
    m = from_sklearn_gbr(est, 5, X)
    Xt, _, _ = _data(42, 2000, 5, 2)
    o = oracle.run(m, Xt)
    leaves = est.apply(Xt).reshape(len(Xt), -1)
    np.testing.assert_array_equal(o["leaf"], leaves)
    np.testing.assert_allclose(o["pred"][:, 0], est.predict(Xt), rtol=1e-5, atol=1e-6)


def test_gradient_boosting_classifier_multiclass_softmax():
    # multiclass boosting (reading c15): K trees per round, softmax probabilities
    X, y, _ = _data(51, 3000, 6, 4)
    est = GradientBoostingClassifier(n_estimators=20, max_depth=3, learning_rate=0.2,
                                     random_state=0).fit(X, y)
    m = from_sklearn_gbc_multiclass(est, 6, X)
    Xt, _, _ = _data(52, 2000, 6, 4)
    o = oracle.run(m, Xt)
    leaves = est.apply(Xt)  # [n, stages, K]
    np.testing.assert_array_equal(o["leaf"], leaves.reshape(len(Xt), -1))
    np.testing.assert_allclose(o["s"], est.decision_function(Xt), rtol=1e-5, atol=1e-6)
    p = est.predict_proba(Xt)
    np.testing.assert_allclose(o["proba"], p, rtol=1e-5, atol=1e-6)
    _check_labels(p, o["label"])

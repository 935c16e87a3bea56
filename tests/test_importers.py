"""Importers (paper_2405_12491_b200/importers.py): model
formats mapped onto the ABI's x <= t / missing_left rule, pinned through the
oracle against hand-computed predictions in the source format's own semantics
(XGBoost x < c, LightGBM NaN-as-zero / NaN-default), and against scikit-learn's
own predictions."""
import numpy as np
import pytest

import oracle
from paper_2405_12491_b200 import importers as I
from synth import gen_x, inject_specials
from tests.helpers import load_golden, parse_x


def test_xgboost_binary_logistic_strict_less_and_default_left():
    g = load_golden("xgboost_binary_logistic.json")
    m = I.from_xgboost_json(g["model"])
    o = oracle.run(m, parse_x(g["X"]))
    np.testing.assert_array_equal(o["s"][:, 0], np.asarray(g["expected"]["margin"]))
    assert o["label"].tolist() == g["expected"]["label"]
    np.testing.assert_allclose(o["proba"][:, 1], g["expected"]["p1"], rtol=1e-6)


def test_xgboost_dart_weight_drop():
    """DART boosters scale each tree's output by weight_drop[i] at
    inference.  Same two trees as xgboost_binary_logistic.json with weights
    (0.5, 2.0); margins by hand: r0 0.5*0.4 + 2*0.25 = 0.7, r1 0.5*0.3 + 2*0.25
    = 0.65, r2 0.5*(-0.2) + 2*0.25 = 0.4, r3 0.5*0.3 + 2*(-0.1) = -0.05."""
    import copy
    g = load_golden("xgboost_binary_logistic.json")
    d = copy.deepcopy(g["model"])
    gb = d["learner"]["gradient_booster"]
    d["learner"]["gradient_booster"] = {"name": "dart", "gbtree": {"name": "gbtree", "model": gb["model"]},
                                        "weight_drop": [0.5, 2.0]}
    m = I.from_xgboost_json(d)
    o = oracle.run(m, parse_x(g["X"]))
    np.testing.assert_allclose(o["s"][:, 0], [0.7, 0.65, 0.4, -0.05], rtol=1e-6, atol=1e-7)
    assert o["label"].tolist() == [1, 1, 1, 0]
    d["learner"]["gradient_booster"]["weight_drop"] = [1.0]
    with pytest.raises(ValueError):
        I.from_xgboost_json(d)


def test_lightgbm_unhandled_output_transforms_rejected():
    import copy
    g = load_golden("lightgbm_binary_dump.json")
    d = copy.deepcopy(g["model"])
    d["objective"] = "regression sqrt"
    with pytest.raises(ValueError):
        I.from_lightgbm_json(d)
    d = copy.deepcopy(g["model"])
    d["objective"], d["average_output"] = "binary sigmoid:2", True
    with pytest.raises(ValueError):
        I.from_lightgbm_json(d)


def test_xgboost_multiclass_softprob():
    g = load_golden("xgboost_multiclass_softprob.json")
    m = I.from_xgboost_json(g["model"])
    assert m.post == I.POST_SOFTMAX and m.tree_output.tolist() == [0, 1, 2]
    o = oracle.run(m, parse_x(g["X"]))
    np.testing.assert_array_equal(o["s"], np.asarray(g["expected"]["margin"]))
    assert o["label"].tolist() == g["expected"]["label"]
    np.testing.assert_allclose(o["proba"], np.asarray(g["expected"]["proba"]), rtol=1e-6)


def test_xgboost_threshold_mapping_is_exact_for_every_fp32():
    # x < c  <=>  x <= nextafter(c, -inf): checked on c's neighbourhood and specials
    cs = np.array([0.5, -0.0, 0.0, 1e-38, -3.25, 1e30, np.float32(1.4e-45)], np.float32)
    thr = np.nextafter(cs, np.float32(-np.inf))
    for c, t in zip(cs, thr):
        xs = np.array([c, np.nextafter(c, np.float32(np.inf)), np.nextafter(c, np.float32(-np.inf)),
                       -np.inf, np.inf, 0.0, -0.0], np.float32)
        np.testing.assert_array_equal(xs < c, xs <= t)


def test_lightgbm_binary_dump_nan_as_zero_and_double_threshold():
    g = load_golden("lightgbm_binary_dump.json")
    m = I.from_lightgbm_json(g["model"])
    o = oracle.run(m, parse_x(g["X"]))
    np.testing.assert_array_equal(o["s"][:, 0], np.asarray(g["expected"]["score"]))
    assert o["label"].tolist() == g["expected"]["label"]
    np.testing.assert_allclose(o["proba"][:, 1], g["expected"]["p1"], rtol=1e-6)


def test_lightgbm_zero_missing_type_rejected_when_not_representable():
    g = load_golden("lightgbm_binary_dump.json")
    d = g["model"]
    root = d["tree_info"][0]["tree_structure"]
    root["missing_type"], root["default_left"] = "Zero", False   # 0 <= 0.1 goes left, default right
    with pytest.raises(ValueError):
        I.from_lightgbm_json(d)
    root["default_left"] = True                                   # agrees with 0.0's comparison
    I.from_lightgbm_json(d)


sk = pytest.importorskip("sklearn")


def _xy(seed, n, F, k):
    X = gen_x(seed, 0, n, F)
    z = X @ np.linspace(-1, 1, F).astype(np.float32)
    return X, np.digitize(z, np.quantile(z, np.linspace(0, 1, k + 1)[1:-1])), z


@pytest.mark.parametrize("kind", ["dt", "rf", "et", "gbr", "gbc2", "gbc4", "rfr"])
def test_from_sklearn_matches_sklearn(kind):
    from sklearn import ensemble as E, tree as Tr
    X, y, z = _xy(91, 2000, 6, 4 if kind == "gbc4" else 2 if kind == "gbc2" else 3)
    X[::37, 2] = np.nan
    est = {"dt": lambda: Tr.DecisionTreeClassifier(max_depth=9, random_state=0),
           "rf": lambda: E.RandomForestClassifier(n_estimators=12, max_depth=7, random_state=0),
           "et": lambda: E.ExtraTreesClassifier(n_estimators=12, max_depth=7, random_state=0),
           "gbr": lambda: E.GradientBoostingRegressor(n_estimators=15, max_depth=3, random_state=0),
           "gbc2": lambda: E.GradientBoostingClassifier(n_estimators=15, max_depth=3, random_state=0),
           "gbc4": lambda: E.GradientBoostingClassifier(n_estimators=15, max_depth=3, random_state=0),
           "rfr": lambda: E.RandomForestRegressor(n_estimators=8, max_depth=6, random_state=0)}[kind]()
    if kind.startswith("gb"):  # sklearn's GradientBoosting does not accept NaN
        X[np.isnan(X)] = 0.0
    est.fit(X, z if kind in ("gbr", "rfr") else y)
    m = I.from_sklearn(est, X)
    Xt = inject_specials(gen_x(92, 0, 1500, 6), 92, rate=0.01 if not kind.startswith("gb") else 0.0)
    Xt[np.isinf(Xt)] = 0.0
    o = oracle.run(m, Xt)
    if kind in ("gbr", "rfr"):
        np.testing.assert_allclose(o["pred"][:, 0], est.predict(Xt), rtol=1e-5, atol=1e-6)
    else:
        np.testing.assert_allclose(o["proba"], est.predict_proba(Xt), rtol=1e-5, atol=1e-6)
    leaves = est.apply(Xt).reshape(len(Xt), -1)
    np.testing.assert_array_equal(o["leaf"], leaves)

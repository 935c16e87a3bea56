"""Oracle pinned to worked examples (tests/golden/, each file cites its passage)."""
import numpy as np
import pytest

import oracle
from synth.trees import stump_model
from tests.helpers import load_golden, model_from_json, model_from_trees, parse_x


def test_spec_288_depth2_tree():
    g = load_golden("spec_288_depth2_tree.json")
    o = oracle.run(model_from_json(g["model"]), parse_x(g["X"]))
    assert o["label"].tolist() == g["expected"]["label"]
    assert o["leaf"].tolist() == g["expected"]["leaf"]
    np.testing.assert_array_equal(o["proba"], np.asarray(g["expected"]["proba"], np.float32))


def test_spec_286_binarizer_as_stumps():
    g = load_golden("spec_286_binarizer_stumps.json")
    X = parse_x(g["X"])
    cols = []
    for st in g["stumps"]:
        m = stump_model(st["feature"], np.float32(st["threshold"]), X.shape[1],
                        st["left_value"], st["right_value"])
        cols.append(oracle.run(m, X)["pred"][:, 0])
    np.testing.assert_array_equal(np.stack(cols, 1), np.asarray(g["expected"]["pred"], np.float32))


def test_spec_287_zero_margin_label_zero():
    g = load_golden("spec_287_zero_margin.json")
    o = oracle.run(model_from_json(g["model"]), parse_x(g["X"]))
    assert o["label"].tolist() == g["expected"]["label"]
    np.testing.assert_array_equal(o["proba"], np.asarray(g["expected"]["proba"], np.float32))


@pytest.mark.parametrize("variant", ["no_missing", "with_missing"])
def test_iris_depth3_hand_tree(variant):
    g = load_golden("iris_depth3_hand.json")
    X = parse_x(g["X"])
    e = g["expected"][variant]
    ml = variant == "with_missing"
    dt = model_from_trees(g["trees"][:1], 4, 3, ml, task=1, agg=0)
    rf = model_from_trees(g["trees"], 4, 3, ml, task=1, agg=0)
    o = oracle.run(dt, X)
    assert o["leaf"][:, 0].tolist() == e["dt_leaf"]
    assert o["label"].tolist() == e["dt_label"]
    o = oracle.run(rf, X)
    assert o["leaf"].tolist() == e["rf_leaf"]
    assert o["label"].tolist() == e["rf_label"]
    np.testing.assert_array_equal(o["proba"], np.asarray(e["rf_proba"], np.float32))


def test_gbdt_two_stumps_hand():
    g = load_golden("gbdt_two_stumps_hand.json")
    X = parse_x(g["X"])
    m = model_from_json(g["model"])
    o = oracle.run(m, X)
    np.testing.assert_array_equal(o["acc"][:, 0], np.asarray(g["expected"]["acc"]))
    np.testing.assert_array_equal(o["pred"][:, 0], np.asarray(g["expected"]["pred"], np.float32))
    m.task, m.post = 1, 1
    o = oracle.run(m, X)
    assert o["label"].tolist() == g["expected"]["label"]
    np.testing.assert_allclose(o["proba"][:, 1], g["expected"]["p1"], rtol=1e-7)
    np.testing.assert_allclose(o["proba"][:, 0], 1 - np.asarray(g["expected"]["p1"]), rtol=1e-6)


def test_gbdt_multiclass_softmax_hand():
    g = load_golden("gbdt_multiclass_softmax_hand.json")
    X = parse_x(g["X"])
    o = oracle.run(model_from_json(g["model"]), X)
    np.testing.assert_array_equal(o["acc"], np.asarray(g["expected"]["acc"]))
    np.testing.assert_array_equal(o["s"], np.asarray(g["expected"]["s"]))
    assert o["label"].tolist() == g["expected"]["label"]
    np.testing.assert_allclose(o["proba"], np.asarray(g["expected"]["proba"]), rtol=1e-6)
    np.testing.assert_allclose(o["proba"].sum(axis=1), 1.0, rtol=1e-6)


def test_multiclass_softmax_golden_matches_its_generator():
    """The fixture's proba block is exactly what the committed generator
    (tests/golden/gen_gbdt_multiclass_softmax.py: math.exp softmax of the
    hand-computed margins) produces."""
    import importlib.util
    import os
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "gen_gbdt_multiclass_softmax.py")
    spec = importlib.util.spec_from_file_location("gen_softmax", path)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    g = load_golden("gbdt_multiclass_softmax_hand.json")
    assert mod.softmax_rows(g["expected"]["s"]) == g["expected"]["proba"]

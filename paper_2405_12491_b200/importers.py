"""Model importers (the paper's `from_sklearn` frontend,
PAPER.md:707): scikit-learn estimators, XGBoost JSON models and LightGBM
``dump_model()`` dicts -> the node-array form of the C ABI (bridger_model_desc,
include/bridger.h).  Host-side argument preparation only: nothing here
predicts.

Split semantics are mapped EXACTLY onto the ABI's "x <= t goes left, NaN goes
to missing_left" rule (readings c1, c2, c4) for fp32 inputs:

* scikit-learn: x <= t64 -> left; t64 rounded toward -inf to fp32
  (x32 <= t64  <=>  x32 <= rd32(t64)); NaN -> missing_go_to_left.
* XGBoost: x < c -> left (c is fp32); x < c  <=>  x <= nextafter(c, -inf) for
  every fp32 x; NaN -> default_left.
* LightGBM: x <= t64 -> left (rounded toward -inf as for sklearn);
  missing_type "NaN": NaN -> default_left; "None": NaN is treated as 0.0, so it
  goes where 0.0 goes (missing_left = [0 <= t]); "Zero": zeros and NaN take the
  default direction -- representable only when that agrees with 0.0's own
  comparison, otherwise ValueError.

Aggregation / post-transform: RF and DT -> MEAN of class fractions; boosting ->
SUM (base + leaf_scale * sum), sigmoid for binary logistic objectives, softmax
with per-tree output indices for multiclass (reading c15).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

TASK_REGRESSION, TASK_CLASSIFICATION = 0, 1
AGG_MEAN, AGG_SUM = 0, 1
POST_IDENTITY, POST_SIGMOID, POST_SOFTMAX = 0, 1, 2


@dataclass
class Ensemble:
    """Arrays of a bridger_model_desc (field names as in include/bridger.h)."""
    n_features: int
    n_outputs: int
    tree_offsets: np.ndarray
    feature: np.ndarray
    threshold: np.ndarray
    left: np.ndarray
    right: np.ndarray
    value: np.ndarray
    task: int = TASK_REGRESSION
    agg: int = AGG_MEAN
    post: int = POST_IDENTITY
    missing_left: Optional[np.ndarray] = None
    base_score: Optional[np.ndarray] = None
    leaf_scale: float = 1.0
    tree_output: Optional[np.ndarray] = None
    classes: Optional[np.ndarray] = None  # label -> class name (caller-side mapping, reading c8)
    meta: dict = field(default_factory=dict)

    @property
    def n_trees(self) -> int:
        return len(self.tree_offsets) - 1


def round_down_f32(t64) -> np.ndarray:
    """Largest fp32 <= t (reading c4): x32 <= t64  <=>  x32 <= round_down_f32(t64)."""
    t64 = np.asarray(t64, np.float64)
    t32 = t64.astype(np.float32)
    over = t32.astype(np.float64) > t64
    t32[over] = np.nextafter(t32[over], np.float32(-np.inf))
    return t32


def _pack(trees, n_features, n_outputs, **kw) -> Ensemble:
    """trees: list of dicts with feature/threshold(fp32)/left/right/value/missing_left."""
    offs = np.zeros(len(trees) + 1, np.int64)
    offs[1:] = np.cumsum([len(t["left"]) for t in trees])
    cat = lambda k, dt: np.concatenate([np.asarray(t[k], dt).reshape(-1) for t in trees])
    has_ml = any(t.get("missing_left") is not None for t in trees)
    ml = None
    if has_ml:
        ml = np.concatenate([np.asarray(t["missing_left"], np.uint8) if t.get("missing_left") is not None
                             else np.zeros(len(t["left"]), np.uint8) for t in trees])
    return Ensemble(n_features=int(n_features), n_outputs=int(n_outputs), tree_offsets=offs,
                    feature=cat("feature", np.int32), threshold=cat("threshold", np.float32),
                    left=cat("left", np.int32), right=cat("right", np.int32), value=cat("value", np.float32),
                    missing_left=ml, **kw)


# ------------------------------------------------------------ scikit-learn --
def _sk_tree(tr, value, with_missing):
    leaf = tr.children_left == -1
    return dict(feature=np.where(leaf, 0, tr.feature).astype(np.int32),
                threshold=np.where(leaf, np.float32(0), round_down_f32(tr.threshold)).astype(np.float32),
                left=tr.children_left.astype(np.int32), right=tr.children_right.astype(np.int32),
                value=np.asarray(value, np.float32),
                missing_left=np.asarray(tr.missing_go_to_left, np.uint8)
                if with_missing and hasattr(tr, "missing_go_to_left") else None)


def _fractions(tr):
    v = tr.value[:, 0, :].astype(np.float64)
    return v / np.maximum(v.sum(axis=1, keepdims=True), 1e-300)


def from_sklearn(est, X_init: Optional[np.ndarray] = None) -> Ensemble:
    """DecisionTree{Classifier,Regressor}, ExtraTree*, RandomForest*, ExtraTrees*,
    GradientBoosting{Classifier,Regressor} (fitted).  Boosting needs one input
    row (X_init) to evaluate the init estimator's constant raw prediction."""
    name = type(est).__name__
    F = int(est.n_features_in_)
    with_missing = True  # sklearn >= 1.3 stores missing_go_to_left (0 where no NaN was seen)
    if name.startswith("GradientBoosting"):
        if X_init is None:
            X_init = np.zeros((1, F))
        init = np.asarray(est._raw_predict_init(np.asarray(X_init[:1], np.float64)), np.float64).reshape(-1)
        S, K = est.estimators_.shape
        trees = [_sk_tree(est.estimators_[s, k].tree_, est.estimators_[s, k].tree_.value[:, 0, 0], with_missing)
                 for s in range(S) for k in range(K)]
        lr = float(est.learning_rate)
        if name == "GradientBoostingRegressor":
            return _pack(trees, F, 1, task=TASK_REGRESSION, agg=AGG_SUM, base_score=init, leaf_scale=lr)
        classes = np.asarray(est.classes_)
        if K == 1:  # binary log-loss: one tree per stage, sigmoid
            return _pack(trees, F, 1, task=TASK_CLASSIFICATION, agg=AGG_SUM, post=POST_SIGMOID,
                         base_score=init, leaf_scale=lr, classes=classes)
        return _pack(trees, F, K, task=TASK_CLASSIFICATION, agg=AGG_SUM, post=POST_SOFTMAX, base_score=init,
                     leaf_scale=lr, tree_output=(np.arange(S * K) % K).astype(np.int32), classes=classes)
    ests = list(est.estimators_) if hasattr(est, "estimators_") else [est]
    if hasattr(est, "classes_"):
        classes = np.asarray(est.classes_)
        if classes.ndim != 1:
            raise ValueError("multi-output classifiers are not supported")
        trees = [_sk_tree(e.tree_, _fractions(e.tree_), with_missing) for e in ests]
        return _pack(trees, F, len(classes), task=TASK_CLASSIFICATION, agg=AGG_MEAN, classes=classes)
    K = int(ests[0].tree_.value.shape[1])
    trees = [_sk_tree(e.tree_, e.tree_.value[:, :, 0], with_missing) for e in ests]
    return _pack(trees, F, K, task=TASK_REGRESSION, agg=AGG_MEAN)


# ------------------------------------------------------------------ XGBoost --
def _xgb_float(v) -> float:
    """base_score is a string ("5E-1"; "[5E-1]" in XGBoost >= 2.1) or a number."""
    if isinstance(v, (list, tuple)):
        v = v[0]
    if isinstance(v, str):
        v = v.strip().strip("[]").split(",")[0]
    return float(v)


def from_xgboost_json(model: dict) -> Ensemble:
    """An XGBoost model saved as JSON (``Booster.save_model("m.json")``), loaded
    with json.load.  gbtree boosters with numerical splits; objectives
    reg:squarederror / reg:linear / reg:absoluteerror (identity),
    binary:logistic / binary:logitraw, multi:softprob / multi:softmax."""
    lrn = model["learner"]
    gb = lrn["gradient_booster"]
    if gb.get("name", "gbtree") not in ("gbtree", "dart"):
        raise ValueError(f"unsupported booster {gb.get('name')}")
    gm = gb["model"] if "model" in gb else gb["gbtree"]["model"]
    # DART: at inference every tree's output is multiplied by its weight_drop
    # (fp32 tree weights); folded into the leaf values (one fp32 rounding per
    # leaf, as XGBoost's own weight * leaf product)
    wdrop = None
    if gb.get("name") == "dart":
        wdrop = np.asarray(gb.get("weight_drop", []), np.float32)
        if len(wdrop) != len(gm["trees"]):
            raise ValueError(f"dart booster: {len(wdrop)} weight_drop entries for {len(gm['trees'])} trees")
    mp = lrn["learner_model_param"]
    F = int(mp["num_feature"])
    K = max(1, int(mp.get("num_class", "0")))
    objective = lrn.get("objective", {}).get("name", "reg:squarederror")
    base = _xgb_float(mp.get("base_score", "0.5"))
    trees = []
    for ti, tj in enumerate(gm["trees"]):
        lc = np.asarray(tj["left_children"], np.int64)
        rc = np.asarray(tj["right_children"], np.int64)
        if any(int(s) != 0 for s in tj.get("split_type", [])):
            raise ValueError("categorical splits are not supported")
        cond = np.asarray(tj["split_conditions"], np.float32)
        leaf = lc == -1
        thr = np.nextafter(cond, np.float32(-np.inf)).astype(np.float32)  # x < c  <=>  x <= prev(c)
        if np.any(~leaf & (cond == np.float32(-np.inf))):
            raise ValueError("split condition -inf is not representable")
        trees.append(dict(feature=np.where(leaf, 0, np.asarray(tj["split_indices"], np.int64)).astype(np.int32),
                          threshold=np.where(leaf, np.float32(0), thr).astype(np.float32),
                          left=lc.astype(np.int32), right=rc.astype(np.int32),
                          value=np.where(leaf, cond if wdrop is None else (cond * wdrop[ti]).astype(np.float32),
                                         np.float32(0)).astype(np.float32),
                          missing_left=np.asarray(tj["default_left"], np.uint8)))
    T = len(trees)
    if objective in ("binary:logistic", "reg:logistic", "binary:logitraw"):
        # base_score is stored as a probability for logistic objectives (ProbToMargin)
        margin = math.log(base / (1.0 - base)) if objective != "binary:logitraw" else base
        post = POST_SIGMOID if objective != "binary:logitraw" else POST_IDENTITY
        task = TASK_CLASSIFICATION if objective != "reg:logistic" else TASK_REGRESSION
        if task == TASK_REGRESSION:
            raise ValueError("reg:logistic outputs probabilities as regression values; not supported")
        return _pack(trees, F, 1, task=task, agg=AGG_SUM, post=post, base_score=np.array([margin]))
    if objective in ("multi:softprob", "multi:softmax"):
        tinfo = np.asarray(gm.get("tree_info", np.arange(T) % K), np.int32)
        return _pack(trees, F, K, task=TASK_CLASSIFICATION, agg=AGG_SUM, post=POST_SOFTMAX,
                     base_score=np.full(K, base), tree_output=tinfo)
    if objective.startswith("reg:") and objective not in ("reg:gamma", "reg:tweedie"):
        return _pack(trees, F, 1, task=TASK_REGRESSION, agg=AGG_SUM, base_score=np.array([base]))
    raise ValueError(f"unsupported objective {objective}")


# ----------------------------------------------------------------- LightGBM --
def _lgb_tree(node: dict, with_default: list):
    """Flatten a LightGBM tree_structure (nested dict) into preorder node arrays."""
    feat, thr, lc, rc, val, ml = [], [], [], [], [], []

    def visit(n):
        i = len(feat)
        feat.append(0); thr.append(0.0); lc.append(-1); rc.append(-1); val.append(0.0); ml.append(0)
        if "leaf_value" in n or "split_feature" not in n:
            val[i] = float(n.get("leaf_value", 0.0))
            return i
        if n.get("decision_type", "<=") != "<=":
            raise ValueError("categorical splits are not supported")
        t64 = float(n["threshold"])
        mt = str(n.get("missing_type", "None"))
        dl = bool(n.get("default_left", True))
        zero_left = 0.0 <= t64
        if mt == "NaN":
            ml[i] = int(dl)
        elif mt == "None":
            ml[i] = int(zero_left)  # NaN is converted to 0.0 before the comparison
        elif mt == "Zero":
            if dl != zero_left:
                raise ValueError("missing_type Zero with a default direction that disagrees with 0.0's split "
                                 "is not representable")
            ml[i] = int(dl)
        else:
            raise ValueError(f"unknown missing_type {mt}")
        feat[i] = int(n["split_feature"])
        thr[i] = float(round_down_f32(t64))
        lc[i] = visit(n["left_child"])
        rc[i] = visit(n["right_child"])
        return i

    visit(node)
    with_default.append(True)
    return dict(feature=np.asarray(feat, np.int32), threshold=np.asarray(thr, np.float32),
                left=np.asarray(lc, np.int32), right=np.asarray(rc, np.int32), value=np.asarray(val, np.float32),
                missing_left=np.asarray(ml, np.uint8))


def from_lightgbm_json(dump: dict) -> Ensemble:
    """A LightGBM ``Booster.dump_model()`` dict: numerical splits; objectives
    regression*, binary (sigmoid:s folded into leaf_scale), multiclass (softmax),
    average_output (random-forest mode -> MEAN)."""
    F = int(dump["max_feature_idx"]) + 1
    K = int(dump.get("num_class", 1))
    tpi = int(dump.get("num_tree_per_iteration", K))
    obj = str(dump.get("objective", "regression")).split()
    flags = []
    trees = [_lgb_tree(t["tree_structure"], flags) for t in dump["tree_info"]]
    agg = AGG_MEAN if dump.get("average_output", False) else AGG_SUM
    name = obj[0] if obj else "regression"
    # objective flags with an output transform this path does not apply
    if "sqrt" in obj[1:]:
        raise ValueError("LightGBM 'regression sqrt' (sign(x) x^2 output transform) is not supported")
    if name == "binary":
        sig = 1.0
        for o in obj[1:]:
            if o.startswith("sigmoid:"):
                sig = float(o.split(":")[1])
        if agg == AGG_MEAN and sig != 1.0:
            # MEAN finalisation is sum / T (reading c6): leaf_scale would be ignored
            raise ValueError("average_output binary models with sigmoid:s != 1 are not supported")
        return _pack(trees, F, 1, task=TASK_CLASSIFICATION, agg=agg, post=POST_SIGMOID, leaf_scale=sig,
                     base_score=np.zeros(1))
    if name in ("multiclass", "softmax"):
        return _pack(trees, F, K, task=TASK_CLASSIFICATION, agg=agg, post=POST_SOFTMAX, base_score=np.zeros(K),
                     tree_output=(np.arange(len(trees)) % tpi).astype(np.int32))
    if name.startswith("regression") or name in ("huber", "fair", "quantile", "mape"):
        return _pack(trees, F, 1, task=TASK_REGRESSION, agg=agg, base_score=np.zeros(1))
    raise ValueError(f"unsupported objective {dump.get('objective')}")


# ---------------------------------------------------------- linear models --
@dataclass
class Linear:
    """Arrays of a bridger_linear_desc (include/bridger.h)."""
    n_features: int
    n_outputs: int
    coef: np.ndarray                  # [K, F] fp64
    intercept: Optional[np.ndarray] = None
    mean: Optional[np.ndarray] = None  # StandardScaler mean_
    scale: Optional[np.ndarray] = None  # StandardScaler scale_
    task: int = TASK_REGRESSION
    post: int = POST_IDENTITY
    classes: Optional[np.ndarray] = None


def from_sklearn_linear(est) -> Linear:
    """LogisticRegression, SGDClassifier, RidgeClassifier, LinearSVC (classifiers);
    LinearRegression, Ridge, Lasso, ElasticNet, SGDRegressor (regressors); or a
    Pipeline(StandardScaler(), <one of those>).  Coefficients are kept in fp64
    (an fp32-fitted model's coefficients are exact in fp64)."""
    mean = scale = None
    if type(est).__name__ == "Pipeline":
        steps = [s for _, s in est.steps]
        if len(steps) != 2 or type(steps[0]).__name__ != "StandardScaler":
            raise ValueError("only Pipeline(StandardScaler(), linear model) is supported")
        sc, est = steps
        F = int(sc.n_features_in_)
        mean = np.asarray(sc.mean_ if sc.with_mean else np.zeros(F), np.float64)
        scale = np.asarray(sc.scale_ if sc.with_std and sc.scale_ is not None else np.ones(F), np.float64)
    coef = np.atleast_2d(np.asarray(est.coef_, np.float64))
    K, F = coef.shape
    b = np.asarray(np.broadcast_to(np.asarray(est.intercept_, np.float64), (K,)), np.float64)
    if hasattr(est, "classes_"):
        name = type(est).__name__
        proba = name == "LogisticRegression" or (name == "SGDClassifier" and est.loss == "log_loss")
        post = (POST_SIGMOID if K == 1 else POST_SOFTMAX) if proba else POST_IDENTITY
        if proba and K > 1 and name == "SGDClassifier":
            raise ValueError("SGDClassifier(log_loss) multiclass proba is one-vs-rest, not softmax")
        return Linear(F, K, coef, b, mean, scale, TASK_CLASSIFICATION, post, np.asarray(est.classes_))
    return Linear(F, K, coef, b, mean, scale, TASK_REGRESSION, POST_IDENTITY)

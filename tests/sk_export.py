"""scikit-learn -> ModelDesc converter (test-side only; the library never links sklearn).

Thresholds are rounded toward -inf to fp32 (reading c4: x32 <= t64 <=> x32 <= rd32(t64)),
leaf values rounded to nearest fp32 (reading c5).
"""
import numpy as np

from synth.trees import ModelDesc, round_down_f32


def _trees_to_desc(trees, n_features, K, value_fn, with_missing, **kw):
    offs, F_, T_, L_, R_, V_, M_ = [0], [], [], [], [], [], []
    for tr in trees:
        n = tr.node_count
        offs.append(offs[-1] + n)
        F_.append(np.where(tr.children_left == -1, 0, tr.feature).astype(np.int32))
        T_.append(np.where(tr.children_left == -1, 0.0, round_down_f32(tr.threshold.astype(np.float64))).astype(np.float32))
        L_.append(tr.children_left.astype(np.int32))
        R_.append(tr.children_right.astype(np.int32))
        V_.append(value_fn(tr).astype(np.float32).reshape(-1))
        M_.append(np.asarray(tr.missing_go_to_left, np.uint8) if with_missing else None)
    return ModelDesc(n_features=n_features, n_outputs=K, tree_offsets=np.asarray(offs, np.int64),
                     feature=np.concatenate(F_), threshold=np.concatenate(T_),
                     left=np.concatenate(L_), right=np.concatenate(R_), value=np.concatenate(V_),
                     missing_left=np.concatenate(M_) if with_missing else None, **kw)


def _class_fractions(tr):
    v = tr.value[:, 0, :].astype(np.float64)
    return v / np.maximum(v.sum(axis=1, keepdims=True), 1e-300)


def from_sklearn_forest(est, n_features, with_missing=False):
    trees = [e.tree_ for e in est.estimators_] if hasattr(est, "estimators_") else [est.tree_]
    K = len(est.classes_)
    return _trees_to_desc(trees, n_features, K, _class_fractions, with_missing, task=1, agg=0)


def from_sklearn_gbr(est, n_features, X_for_init):
    trees = [e[0].tree_ for e in est.estimators_]
    init = float(np.asarray(est._raw_predict_init(X_for_init[:1].astype(np.float64))).reshape(-1)[0])
    return _trees_to_desc(trees, n_features, 1, lambda tr: tr.value[:, 0, 0], False,
                          task=0, agg=1, base_score=np.array([init]), leaf_scale=float(est.learning_rate))


def from_sklearn_gbc_multiclass(est, n_features, X_for_init):
    """GradientBoostingClassifier with K >= 3 classes: estimators_[stage, k] is the
    class-k regression tree of a round; raw = init + lr * sum (predict_stages),
    proba = softmax(raw) (reading c15).  Trees are laid out round-major, so tree
    t = stage t // K adds to output t % K."""
    S, K = est.estimators_.shape
    trees = [est.estimators_[s, k].tree_ for s in range(S) for k in range(K)]
    init = np.asarray(est._raw_predict_init(X_for_init[:1].astype(np.float64)), np.float64).reshape(-1)
    return _trees_to_desc(trees, n_features, K, lambda tr: tr.value[:, 0, 0], False,
                          task=1, agg=1, post=2, base_score=init, leaf_scale=float(est.learning_rate),
                          tree_output=(np.arange(S * K) % K).astype(np.int32))

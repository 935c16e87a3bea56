"""Seeded tree ensembles in the C-ABI node-array form.

A ``ModelDesc`` holds, for T trees concatenated:
  tree_offsets int64[T+1]   node range of each tree (tree-local ids inside)
  feature      int32[n]     split feature (ignored at leaves)
  threshold    float32[n]   go LEFT iff x <= threshold
  left, right  int32[n]     tree-local child ids, both -1 at leaves, root = 0
  value        float32[n*K] read at leaves only
  missing_left uint8[n] | None   NaN routing per node (None => NaN goes right)
  tree_output  int32[T] | None   multiclass boosting: tree t adds its SCALAR leaf
                                 values (value float32[n]) to output tree_output[t]
plus task / agg / post / base_score / leaf_scale.

Thresholds are *calibrated* like a trainer would place them:
a calibration sample from the same X generator is split top-down; each node
takes a random feature and the midpoint of two adjacent sorted values at a
random quantile in [0.25, 0.75] of the rows reaching it, rounded toward -inf to
fp32 (reading c4).  This is tree *construction*; nothing here predicts.
"""
from __future__ import annotations

from dataclasses import dataclass, field, replace
from typing import Optional

import numpy as np

from .xgen import gen_x, splitmix64_np, _seed_key

TASK_REGRESSION, TASK_CLASSIFICATION = 0, 1
AGG_MEAN, AGG_SUM = 0, 1
POST_IDENTITY, POST_SIGMOID, POST_SOFTMAX = 0, 1, 2


@dataclass
class ModelDesc:
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
    meta: dict = field(default_factory=dict)
    tree_output: Optional[np.ndarray] = None

    @property
    def value_width(self) -> int:
        """Values stored per node: 1 with tree_output (scalar leaves), else K."""
        return 1 if self.tree_output is not None else self.n_outputs

    @property
    def n_trees(self) -> int:
        return len(self.tree_offsets) - 1

    @property
    def n_nodes(self) -> int:
        return int(self.tree_offsets[-1])

    def tree(self, t: int):
        a, b = int(self.tree_offsets[t]), int(self.tree_offsets[t + 1])
        K = self.value_width
        return dict(feature=self.feature[a:b], threshold=self.threshold[a:b],
                    left=self.left[a:b], right=self.right[a:b],
                    value=self.value[a * K:b * K].reshape(b - a, K),
                    missing_left=None if self.missing_left is None else self.missing_left[a:b])

    def subset(self, trees) -> "ModelDesc":
        """Model made of the listed trees (in that order); used for tree sharding."""
        trees = list(trees)
        parts = [self.tree(t) for t in trees]
        sizes = [len(p["feature"]) for p in parts]
        offs = np.zeros(len(trees) + 1, dtype=np.int64)
        offs[1:] = np.cumsum(sizes)
        cat = lambda k: np.concatenate([p[k] for p in parts]) if parts else np.zeros(0)
        return replace(
            self, tree_offsets=offs,
            feature=cat("feature").astype(np.int32), threshold=cat("threshold").astype(np.float32),
            left=cat("left").astype(np.int32), right=cat("right").astype(np.int32),
            value=np.concatenate([p["value"].reshape(-1) for p in parts]).astype(np.float32),
            missing_left=None if self.missing_left is None else cat("missing_left").astype(np.uint8),
            tree_output=None if self.tree_output is None else np.asarray(self.tree_output, np.int32)[trees],
            meta=dict(self.meta))


def _hash_u64(seed: int, *ints) -> np.ndarray:
    """Counter hash: splitmix64(key(seed) + mixed counters), vectorised over arrays."""
    key = np.uint64(_seed_key(seed))
    acc = np.zeros(np.broadcast(*[np.asarray(i) for i in ints]).shape if ints else (), dtype=np.uint64)
    with np.errstate(over="ignore"):
        for i in ints:
            acc = splitmix64_np(acc ^ np.asarray(i, dtype=np.uint64))
        return splitmix64_np(acc + key)


def _unit(h: np.ndarray) -> np.ndarray:
    return (h >> np.uint64(11)).astype(np.float64) * (1.0 / (1 << 53))


def round_down_f32(v64: np.ndarray) -> np.ndarray:
    """Largest fp32 <= v (reading c4: exact for every fp32 x)."""
    t = v64.astype(np.float32)
    bad = t.astype(np.float64) > v64
    t[bad] = np.nextafter(t[bad], np.float32(-np.inf))
    return t


def _leaf_values(seed, n_trees, n_leaves, K, kind, lr):
    t = np.arange(n_trees, dtype=np.uint64)[:, None, None]
    l = np.arange(n_leaves, dtype=np.uint64)[None, :, None]
    k = np.arange(K, dtype=np.uint64)[None, None, :]
    if kind == "classification":
        c = (_hash_u64(seed, t, l, k) >> np.uint64(32)).astype(np.int64) % 65  # U{0..64}
        n = c.sum(axis=2, keepdims=True)
        c[..., :1] += (n == 0)
        n = c.sum(axis=2, keepdims=True)
        return (c.astype(np.float64) / n.astype(np.float64)).astype(np.float32)
    # regression: lr * z, z Irwin-Hall on the same 2^-19 lattice as X
    s = np.zeros((n_trees, n_leaves, K), dtype=np.int64)
    for j in range(4):
        s += (_hash_u64(seed, t, l, k, np.uint64(j)) >> np.uint64(44)).astype(np.int64)
    z = (s - (1 << 21)).astype(np.float64) * 2.0 ** -19
    return (np.float32(lr) * z.astype(np.float32)).astype(np.float32)


def perfect_ensemble(seed: int, n_trees: int, depth: int, n_features: int, *,
                     kind: str = "regression", n_classes: int = 1, agg: Optional[int] = None,
                     post: int = POST_IDENTITY, lr: float = 0.1, base_score=None,
                     calib_rows: int = 4096, x_seed: Optional[int] = None,
                     calib_x: Optional[np.ndarray] = None) -> ModelDesc:
    """T perfect trees of depth D in heap order (children of i: 2i+1, 2i+2).

    kind="classification": K = n_classes, leaf values are class fractions c_k/n
    with c_k ~ U{0..64} (MEAN aggregation, RF/DT style).
    kind="regression": K = 1, leaf values lr*z (SUM aggregation, GBDT style,
    base_score default 0.5) unless agg says otherwise.
    """
    T, D, F = n_trees, depth, n_features
    I, L = (1 << D) - 1, 1 << D
    K = n_classes if kind == "classification" else 1
    if x_seed is None:
        x_seed = seed
    if calib_x is None:
        rows = int(max(256, min(calib_rows, (1 << 25) // max(T, 1))))
        Xc = gen_x(x_seed ^ 0xCA11B, 0, rows, F)
    else:
        Xc = np.asarray(calib_x, dtype=np.float32)
        rows = Xc.shape[0]
    # dense per-column ranks of the calibration sample + the sorted unique values
    uniq, codes = [], np.empty((rows, F), dtype=np.int64)
    for c in range(F):
        u, inv = np.unique(Xc[:, c].astype(np.float64), return_inverse=True)
        uniq.append(u)
        codes[:, c] = inv
    width = max(len(u) for u in uniq)
    utab = np.zeros((F, width), dtype=np.float64)
    for c, u in enumerate(uniq):
        utab[c, :len(u)] = u

    feat = np.zeros((T, max(I, 1)), dtype=np.int32)
    thr = np.zeros((T, max(I, 1)), dtype=np.float32)
    pos = np.zeros((T, rows), dtype=np.int64)            # heap position of each calib row
    tt = np.arange(T, dtype=np.int64)[:, None]
    for lvl in range(D):
        lo, n_lvl = (1 << lvl) - 1, 1 << lvl
        nodes = np.arange(lo, lo + n_lvl, dtype=np.uint64)
        hf = _hash_u64(seed, np.arange(T, dtype=np.uint64)[:, None], nodes[None, :], np.uint64(1))
        f_lvl = ((hf >> np.uint64(20)) % np.uint64(F)).astype(np.int32)       # [T, n_lvl]
        q_lvl = 0.25 + 0.5 * _unit(_hash_u64(seed, np.arange(T, dtype=np.uint64)[:, None],
                                               nodes[None, :], np.uint64(2)))
        feat[:, lo:lo + n_lvl] = f_lvl
        local = pos - lo                                                      # [T, rows]
        fr = f_lvl[tt, local]                                                 # feature per (t, row)
        val = codes[np.arange(rows)[None, :], fr]                             # [T, rows]
        group = tt * n_lvl + local
        key = np.sort((group * (1 << 23) + val).reshape(-1))
        gid = key >> 23
        sval = key & ((1 << 23) - 1)
        cnt = np.bincount(gid, minlength=T * n_lvl)
        start = np.concatenate([[0], np.cumsum(cnt)[:-1]])
        q = q_lvl.reshape(-1)
        k = np.floor(q * (np.maximum(cnt, 2) - 2)).astype(np.int64)
        ok = cnt >= 2
        a = np.where(ok, sval[np.minimum(start + k, len(sval) - 1)], 0)
        b = np.where(ok, sval[np.minimum(start + k + 1, len(sval) - 1)], 0)
        fg = f_lvl.reshape(-1)
        mid = (utab[fg, a] + utab[fg, b]) * 0.5
        # fallback: a random lattice value in [-1, 1)
        hfb = _hash_u64(seed, np.arange(T * n_lvl, dtype=np.uint64), np.uint64(3))
        fb = ((hfb >> np.uint64(44)).astype(np.int64) - (1 << 19)) * 2.0 ** -19
        t_lvl = round_down_f32(np.where(ok, mid, fb)).reshape(T, n_lvl)
        thr[:, lo:lo + n_lvl] = t_lvl
        # split the calibration rows (construction)
        x_at = Xc[np.arange(rows)[None, :], fr]
        go_right = x_at > t_lvl[tt, local]
        pos = 2 * pos + 1 + go_right

    vals = _leaf_values(seed ^ 0x1EAF, T, L, K, kind, lr)                    # [T, L, K]
    n_nodes = I + L
    feature = np.zeros((T, n_nodes), dtype=np.int32)
    threshold = np.zeros((T, n_nodes), dtype=np.float32)
    left = np.full((T, n_nodes), -1, dtype=np.int32)
    right = np.full((T, n_nodes), -1, dtype=np.int32)
    value = np.zeros((T, n_nodes, K), dtype=np.float32)
    if I:
        feature[:, :I] = feat[:, :I]
        threshold[:, :I] = thr[:, :I]
        ii = np.arange(I, dtype=np.int32)
        left[:, :I] = 2 * ii + 1
        right[:, :I] = 2 * ii + 2
    value[:, I:, :] = vals
    if agg is None:
        agg = AGG_MEAN if kind == "classification" else AGG_SUM
    task = TASK_CLASSIFICATION if kind == "classification" else TASK_REGRESSION
    if agg == AGG_SUM and base_score is None:
        base_score = np.full(K, 0.5)
    offs = np.arange(T + 1, dtype=np.int64) * n_nodes
    return ModelDesc(n_features=F, n_outputs=K, tree_offsets=offs,
                     feature=feature.reshape(-1), threshold=threshold.reshape(-1),
                     left=left.reshape(-1), right=right.reshape(-1), value=value.reshape(-1),
                     task=task, agg=agg, post=post,
                     base_score=None if base_score is None else np.asarray(base_score, np.float64),
                     leaf_scale=1.0, meta=dict(seed=seed, depth=D, kind=kind))


def prune_ensemble(m: ModelDesc, seed: int, p: float = 0.1, with_missing: bool = False) -> ModelDesc:
    """Correctness variant: each internal non-root node becomes a leaf with
    probability p (its subtree dropped); nodes are renumbered in DFS preorder
    (sklearn's order), so the result is non-perfect and not in heap order.
    with_missing=True adds a random per-node ``missing_left`` array."""
    K = m.value_width
    out_f, out_t, out_l, out_r, out_v, out_m, offs = [], [], [], [], [], [], [0]
    for t in range(m.n_trees):
        tr = m.tree(t)
        new_ids = {}
        order = []
        stack = [(0, 0)]
        while stack:
            n, d = stack.pop()
            h = _unit(_hash_u64(seed, np.uint64(t), np.uint64(n)))
            is_leaf = tr["left"][n] == -1 or (d > 0 and float(h) < p)
            new_ids[n] = len(order)
            order.append((n, is_leaf))
            if not is_leaf:
                stack.append((int(tr["right"][n]), d + 1))
                stack.append((int(tr["left"][n]), d + 1))
        f = np.zeros(len(order), np.int32); th = np.zeros(len(order), np.float32)
        lf = np.full(len(order), -1, np.int32); rt = np.full(len(order), -1, np.int32)
        v = np.zeros((len(order), K), np.float32); ml = np.zeros(len(order), np.uint8)
        for j, (n, is_leaf) in enumerate(order):
            if is_leaf:
                if tr["left"][n] == -1:
                    v[j] = tr["value"][n]
                else:  # a pruned internal node takes the value of its leftmost leaf
                    c = n
                    while tr["left"][c] != -1:
                        c = int(tr["left"][c])
                    v[j] = tr["value"][c]
            else:
                f[j] = tr["feature"][n]; th[j] = tr["threshold"][n]
                lf[j] = new_ids[int(tr["left"][n])]; rt[j] = new_ids[int(tr["right"][n])]
                ml[j] = int(_hash_u64(seed ^ 0x77, np.uint64(t), np.uint64(n)) & np.uint64(1))
        out_f.append(f); out_t.append(th); out_l.append(lf); out_r.append(rt)
        out_v.append(v.reshape(-1)); out_m.append(ml); offs.append(offs[-1] + len(order))
    return replace(m, tree_offsets=np.asarray(offs, np.int64),
                   feature=np.concatenate(out_f), threshold=np.concatenate(out_t),
                   left=np.concatenate(out_l), right=np.concatenate(out_r),
                   value=np.concatenate(out_v),
                   missing_left=np.concatenate(out_m) if with_missing else None,
                   meta=dict(m.meta, pruned=p))


def stump_model(feature: int, threshold: float, n_features: int, left_value: float,
                right_value: float) -> ModelDesc:
    """Single depth-1 regression tree (SPEC.md:286 binarizer == one stump per column)."""
    return ModelDesc(n_features=n_features, n_outputs=1,
                     tree_offsets=np.array([0, 3], np.int64),
                     feature=np.array([feature, 0, 0], np.int32),
                     threshold=np.array([threshold, 0, 0], np.float32),
                     left=np.array([1, -1, -1], np.int32), right=np.array([2, -1, -1], np.int32),
                     value=np.array([0.0, left_value, right_value], np.float32),
                     task=TASK_REGRESSION, agg=AGG_MEAN, post=POST_IDENTITY)


def multiclass_gbdt(seed: int, n_rounds: int, depth: int, n_features: int, n_classes: int, *,
                    lr: float = 0.1, calib_rows: int = 2048) -> ModelDesc:
    """Multiclass gradient boosting (reading c15): n_rounds x K perfect
    regression trees, tree t = round t // K for class t % K, scalar leaves
    lr*z, SUM aggregation, base_score = per-class log-prior-like constants,
    softmax probabilities."""
    K = int(n_classes)
    m = perfect_ensemble(seed, n_rounds * K, depth, n_features, kind="regression", lr=lr,
                         calib_rows=calib_rows)
    base = np.log(np.arange(1, K + 1, dtype=np.float64) / (K * (K + 1) / 2))
    return replace(m, n_outputs=K, task=TASK_CLASSIFICATION, agg=AGG_SUM, post=POST_SOFTMAX,
                   base_score=base, tree_output=(np.arange(n_rounds * K) % K).astype(np.int32),
                   meta=dict(m.meta, kind="multiclass_gbdt"))

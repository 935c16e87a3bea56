"""Oracle pinned by brute force on tiny inputs (SURVEY.md §8(c) 'walk semantics
(independent computation)').

The region oracle never walks: each leaf's root path is turned into per-feature
interval constraints (x <= t  ->  x in [-inf, t];  x > t  ->  x in (t, +inf];
NaN allowed iff the path's missing directions say so), and every input on the
critical grid {each threshold, nextafter(t, +-inf), +-0, +-inf, NaN, min
subnormal}^F is tested against all leaves at once.  Exactly one leaf must
contain each point, and it must be the oracle's leaf.
"""
import itertools

import numpy as np
import pytest

import oracle
from synth import perfect_ensemble, prune_ensemble


def leaf_regions(tree, n_features):
    """{leaf_id: [(lo, lo_open, hi, hi_open, nan_ok) per feature]} by path enumeration."""
    out = {}
    init = [(-np.inf, False, np.inf, False, True)] * n_features
    stack = [(0, list(init))]
    while stack:
        n, cons = stack.pop()
        if tree["left"][n] == -1:
            out[n] = cons
            continue
        f, t = int(tree["feature"][n]), float(tree["threshold"][n])
        ml = bool(tree["missing_left"][n]) if tree["missing_left"] is not None else False
        lo, lo_o, hi, hi_o, nan_ok = cons[f]
        left = list(cons)
        if t < hi or (t == hi and hi_o):
            left[f] = (lo, lo_o, t, False, nan_ok and ml)
        else:
            left[f] = (lo, lo_o, hi, hi_o, nan_ok and ml)
        right = list(cons)
        if t > lo or (t == lo and not lo_o):
            right[f] = (t, True, hi, hi_o, nan_ok and not ml)
        else:
            right[f] = (lo, lo_o, hi, hi_o, nan_ok and not ml)
        stack.append((int(tree["left"][n]), left))
        stack.append((int(tree["right"][n]), right))
    return out


def contains(cons, x):
    for (lo, lo_o, hi, hi_o, nan_ok), v in zip(cons, x):
        v = float(v)
        if np.isnan(v):
            if not nan_ok:
                return False
            continue
        if v < lo or (v == lo and lo_o) or v > hi or (v == hi and hi_o):
            return False
    return True


def critical_grid(model, n_features, cap=12):
    per = []
    for f in range(n_features):
        internal = model.left != -1
        ts = np.unique(model.threshold[internal & (model.feature == f)])[:cap]
        vals = [np.float32(v) for v in (np.nan, np.inf, -np.inf, 0.0, -0.0, 1.4e-45)]
        for t in ts:
            vals += [t, np.nextafter(t, np.float32(np.inf)), np.nextafter(t, np.float32(-np.inf))]
        per.append(vals)
    return np.array(list(itertools.product(*per)), dtype=np.float32)


@pytest.mark.parametrize("seed,depth,F,p,ml", [
    (11, 1, 1, 0.0, False), (12, 2, 2, 0.0, False), (13, 3, 2, 0.3, False),
    (14, 3, 3, 0.3, True), (15, 4, 2, 0.2, True), (16, 4, 3, 0.0, True),
])
def test_region_bruteforce_matches_walker(seed, depth, F, p, ml):
    m = perfect_ensemble(seed, 3, depth, F, kind="classification", n_classes=2, calib_rows=64)
    m = prune_ensemble(m, seed, p=p, with_missing=ml)
    X = critical_grid(m, F)
    o = oracle.run(m, X, n_threads=2)
    for t in range(m.n_trees):
        tr = m.tree(t)
        regions = leaf_regions(tr, F)
        for r in range(X.shape[0]):
            hits = [l for l, c in regions.items() if contains(c, X[r])]
            assert len(hits) == 1, (t, r, X[r], hits)
            assert hits[0] == o["leaf"][r, t], (t, r, X[r], hits, o["leaf"][r, t])

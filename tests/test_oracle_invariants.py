"""Oracle pinned by invariants that the mathematics fixes:
additivity of raw sums over tree sets, tree-permutation invariance (exact under
condition E: all sums of fp32 leaf values are exact in fp64), T copies of one
tree, row-shard concatenation, thread-count determinism, proba rows summing to 1."""
import numpy as np

import oracle
from synth import gen_x, make_config, perfect_ensemble, prune_ensemble


def _model(kind="classification", K=3, T=40, D=5, F=7, seed=5):
    m = perfect_ensemble(seed, T, D, F, kind=kind, n_classes=K, calib_rows=512)
    return prune_ensemble(m, seed, p=0.15, with_missing=True)


def test_additivity_over_tree_sets():
    m = _model()
    X = gen_x(9, 0, 700, 7)
    full = oracle.run(m, X)["acc"]
    a = oracle.run(m.subset(range(0, 17)), X)["acc"]
    b = oracle.run(m.subset(range(17, m.n_trees)), X)["acc"]
    np.testing.assert_array_equal(full, a + b)


def test_tree_permutation_invariance():
    m = _model(kind="regression", K=1)
    X = gen_x(10, 0, 500, 7)
    perm = np.random.default_rng(0).permutation(m.n_trees)
    o1 = oracle.run(m, X)
    o2 = oracle.run(m.subset(perm), X)
    np.testing.assert_array_equal(o1["acc"], o2["acc"])
    np.testing.assert_array_equal(o1["leaf"][:, perm], o2["leaf"])


def test_copies_of_one_tree():
    m = _model(T=1)
    X = gen_x(11, 0, 300, 7)
    one = oracle.run(m, X)
    rf = oracle.run(m.subset([0] * 13), X)
    np.testing.assert_array_equal(one["proba"], rf["proba"])
    np.testing.assert_array_equal(one["label"], rf["label"])
    g = _model(kind="regression", K=1, T=1)
    one = oracle.run(g, X)["acc"]
    many = oracle.run(g.subset([0] * 13), X)["acc"]
    np.testing.assert_array_equal(many, 13 * one)


def test_row_shards_and_threads():
    _, m = make_config("C2", n_trees=20)
    X = gen_x(2, 0, 1001, 28)
    full = oracle.run(m, X, n_threads=1)
    parts = [oracle.run(m, X[a:b], n_threads=3) for a, b in [(0, 333), (333, 334), (334, 1001)]]
    for k in full:
        np.testing.assert_array_equal(full[k], np.concatenate([p[k] for p in parts]))


def test_proba_rows_sum_to_one_and_leaf_is_leaf():
    m = _model(K=4)
    X = gen_x(12, 0, 400, 7)
    o = oracle.run(m, X)
    np.testing.assert_allclose(o["proba"].sum(1), 1.0, atol=4 * m.n_trees * 2 ** -23)
    offs = m.tree_offsets
    for t in range(m.n_trees):
        assert np.all(m.left[offs[t] + o["leaf"][:, t]] == -1)

"""Parity at BASELINE.json's full sizes, in the launch configurations bench.py
times, checked on seeded row samples the oracle computes one by one
(SURVEY.md §4b.4): C3 (10M x 90, 500 trees), C4's per-GPU slice (12.5M x 64 rows
of the row-sharded 100M, 1000 depth-12 trees, 8 classes) and C5 (10M x 200,
10,000 depth-10 trees, run as 8 tree shards whose exact int64 partials are
summed and finalised -- the tree-sharded data path, on one GPU)."""
import numpy as np
import pytest

import oracle
from paper_2405_12491_b200.dist import TIER_CODE, tree_partition, tree_visits
from synth import gen_x, gen_x_torch, make_config

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
import paper_2405_12491_b200 as B  # noqa: E402


def _sample_rows(n, k=2048, seed=0):
    rows = np.sort(np.random.default_rng(seed).choice(n, k, replace=False))
    return np.unique(np.concatenate([rows, [0, 31, 32, n - 1]]))


def _x_rows(cfg, rows, row0=0):
    return np.concatenate([gen_x(cfg.seed, row0 + int(r), 1, cfg.n_features) for r in rows])


@pytest.mark.parametrize("binning", [None, "entry_lockstep"])
def test_c3_full_size_sampled(binning, monkeypatch):
    """C3 at full size (the bench's launch configuration), and with the
    bucket-entry binning kernel in lockstep epochs (cooperative launch, grid
    barriers every ~24 MB of X: the path for inputs larger than L2)."""
    if binning:
        monkeypatch.setenv("BRIDGER_BIN", "E")
        monkeypatch.setenv("BRIDGER_BIN_LOCK", "1")
    c, m = make_config("C3")
    g = B.Model(m)
    X = gen_x_torch(c.seed, 0, c.n_rows, c.n_features, device="cuda")
    pred = g.predict(X).cpu().numpy()
    del X
    rows = _sample_rows(c.n_rows)
    o = oracle.run(m, _x_rows(c, rows))
    np.testing.assert_array_equal(pred[rows], o["pred"])       # tier E53: bitwise


def test_c4_per_gpu_slice_full_size_sampled():
    c, m = make_config("C4")
    n = c.n_rows // 8                                            # rank 0 of the x8 row sharding
    g = B.Model(m)
    X = gen_x_torch(c.seed, 0, n, c.n_features, device="cuda")
    lab = g.predict(X).cpu().numpy()
    pr = g.predict_proba(X).cpu().numpy()
    del X
    rows = _sample_rows(n, k=1024)
    o = oracle.run(m, _x_rows(c, rows))
    np.testing.assert_array_equal(lab[rows], o["label"])
    np.testing.assert_array_equal(pr[rows], o["proba"])


def test_c5_tree_sharded_full_size_sampled():
    c, m = make_config("C5")
    q, tier, _ = B.analyze_exactness(m)
    X = gen_x_torch(c.seed, 0, c.n_rows, c.n_features, device="cuda")
    acc = torch.zeros((c.n_rows, 1), dtype=torch.int64, device="cuda")
    shards = tree_partition(tree_visits(m), 8)
    g0 = None
    for a, b in shards:                                         # the 8 ranks' work, one after another
        g = B.Model(m.subset(range(a, b)), force_fixed_point=(q, TIER_CODE[tier]))
        acc += g.predict_raw(X)
        g0 = g0 or g
    del X
    pred = g0.finalize(acc, total_trees=m.n_trees).cpu().numpy()
    raw = acc.cpu().numpy()[:, 0]
    rows = _sample_rows(c.n_rows, k=512)
    Xs = _x_rows(c, rows)
    o = oracle.run(m, Xs)
    # exact integer sum of the leaf values the oracle's walk reached
    ints = np.round(np.ldexp(m.value.astype(np.float64), -q)).astype(np.int64)
    exact = np.zeros(len(rows), np.int64)
    for t in range(m.n_trees):
        exact += ints[m.tree_offsets[t] + o["leaf"][:, t]]
    np.testing.assert_array_equal(raw[rows], exact)
    want = (np.float64(0.5) + exact.astype(np.float64) * 2.0 ** q).astype(np.float32)
    np.testing.assert_array_equal(pred[rows, 0], want)
    np.testing.assert_allclose(pred[rows, 0], o["pred"][:, 0], rtol=1e-5, atol=1e-6)

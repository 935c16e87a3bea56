"""CUDA path vs the oracle, element by element, through the C ABI.

Bar (BASELINE.json north_star): labels and leaf indices bit-exact; scores and
probabilities bit-exact under exactness tier E53 (reading c9), else rtol 1e-5;
sigmoid probabilities rtol 1e-5 (reading c10).  Sizes span many 32-row blocks,
several tree chunks and a ragged tail; the full-size C2 run (bench launch
configuration) is checked on a seeded row sample the oracle computes one by one.
"""
import numpy as np
import pytest

import oracle
from synth import gen_x, gen_x_torch, inject_specials, make_config, perfect_ensemble, prune_ensemble
from synth.trees import ModelDesc

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
import paper_2405_12491_b200 as B  # noqa: E402


def dev(X):
    return torch.from_numpy(np.ascontiguousarray(X)).cuda()


def check(m, X, variant=None, exact=True, apply=True):
    g = B.Model(m, variant=variant)
    o = oracle.run(m, X)
    Xd = dev(X)
    torch.cuda.synchronize()
    if m.task == 1:
        lab = g.predict(Xd).cpu().numpy()
        np.testing.assert_array_equal(lab, o["label"])
        pr = g.predict_proba(Xd).cpu().numpy()
        if exact and m.post == 0:
            np.testing.assert_array_equal(pr, o["proba"])
        else:
            np.testing.assert_allclose(pr, o["proba"], rtol=1e-5, atol=1e-7)
    else:
        pred = g.predict(Xd).cpu().numpy()
        if exact:
            np.testing.assert_array_equal(pred, o["pred"])
        else:
            np.testing.assert_allclose(pred, o["pred"], rtol=1e-5, atol=1e-6)
    if apply:
        np.testing.assert_array_equal(g.apply(Xd).cpu().numpy(), o["leaf"])
    info = g.info()
    raw = g.predict_raw(Xd).cpu().numpy()
    a = raw.astype(np.float64) * 2.0 ** info["acc_scale_exp"] if info["acc_is_int64"] else raw
    if exact:
        np.testing.assert_array_equal(a, o["acc"])
    else:
        np.testing.assert_allclose(a, o["acc"], rtol=1e-9, atol=1e-12)
    return g, o


def test_c1_iris_decision_tree():
    c, m = make_config("C1")
    from synth import iris_like_x
    check(m, iris_like_x(1))


@pytest.mark.parametrize("n_rows", [1, 31, 33, 20011])
def test_c2_random_forest_rows(n_rows):
    c, m = make_config("C2")
    check(m, gen_x(2, 0, n_rows, 28), apply=n_rows < 5000)


def test_c3_gbdt_regression():
    c, m = make_config("C3")
    check(m, gen_x(3, 0, 30011, 90))


def test_c5_shaped_deep_wide():
    c, m = make_config("C5", n_trees=24)
    check(m, gen_x(5, 0, 3001, 200))


@pytest.mark.parametrize("ml", [False, True])
def test_pruned_trees_specials_missing(ml):
    m = perfect_ensemble(7, 70, 7, 13, kind="classification", n_classes=5, calib_rows=1024)
    m = prune_ensemble(m, 7, p=0.15, with_missing=ml)
    X = inject_specials(gen_x(8, 0, 5003, 13), 8, rate=0.02)
    check(m, X)


def test_binary_gbdt_sigmoid():
    m = perfect_ensemble(9, 150, 6, 17, kind="regression", lr=0.1)
    m.task, m.post = 1, 1
    check(m, gen_x(10, 0, 4099, 17), exact=False)


def test_f64_tier_tolerance():
    m = perfect_ensemble(11, 40, 5, 9, kind="regression", lr=0.1)
    v = m.value.copy()
    v[np.nonzero(m.left == -1)[0][0]] = np.float32(1.4e-45)      # subnormal leaf -> q = -149 -> F64 tier
    m = ModelDesc(**{**m.__dict__, "value": v})
    assert B.analyze_exactness(m)[1] == "F64"
    check(m, gen_x(12, 0, 2000, 9), exact=False)


def test_zero_rows_and_shape_errors():
    c, m = make_config("C2", n_trees=10)
    g = B.Model(m)
    out = g.predict(torch.empty((0, 28), device="cuda"))
    assert out.shape == (0,)
    bad = torch.zeros((4, 27), device="cuda")
    out4 = torch.zeros(4, dtype=torch.int32, device="cuda")
    with pytest.raises(B.BridgerError) as ei:
        B._check(B.lib().bridger_predict(g._h, bad.data_ptr(), 4, 27, out4.data_ptr(), None))
    assert ei.value.status == B.E_SHAPE
    c3, r = make_config("C3", n_trees=5)
    with pytest.raises(B.BridgerError):
        B.Model(r).predict_proba(torch.zeros((4, 90), device="cuda"))


@pytest.mark.parametrize("codes", ["0", "1"])
def test_predict_host_matches_device(codes, monkeypatch):
    monkeypatch.setenv("BRIDGER_CODES", codes)
    c, m = make_config("C2", n_trees=30)
    X = gen_x(2, 0, 70001, 28)
    g = B.Model(m)
    a = g.predict(dev(X)).cpu().numpy()
    b = g.predict_host(torch.from_numpy(X).pin_memory()).numpy()
    np.testing.assert_array_equal(a, b)
    p = g.predict_host(X, proba=True).numpy()
    np.testing.assert_array_equal(p, g.predict_proba(dev(X)).cpu().numpy())


def test_tree_shards_add_exactly():
    """raw(A) + raw(B) finalised == predict(A u B), bitwise (reading c9, tree sharding)."""
    c, m = make_config("C3", n_trees=120)
    q, tier, _ = B.analyze_exactness(m)
    tiers = {"E53": 0, "E63": 1, "F64": 2}
    X = dev(gen_x(3, 0, 9001, 90))
    full = B.Model(m).predict(X)
    ga = B.Model(m.subset(range(0, 50)), force_fixed_point=(q, tiers[tier]))
    gb = B.Model(m.subset(range(50, 120)), force_fixed_point=(q, tiers[tier]))
    acc = ga.predict_raw(X) + gb.predict_raw(X)
    out = ga.finalize(acc, total_trees=120)
    assert torch.equal(out, full)


def test_c2_full_size_sampled():
    """BASELINE configs[1] at full size in the bench launch configuration;
    a seeded sample of rows is checked against the oracle row by row."""
    c, m = make_config("C2")
    Xd = gen_x_torch(2, 0, c.n_rows, c.n_features, device="cuda")
    g = B.Model(m)
    lab = g.predict(Xd).cpu().numpy()
    pr = g.predict_proba(Xd).cpu().numpy()
    rows = np.sort(np.random.default_rng(0).choice(c.n_rows, 4096, replace=False))
    rows = np.unique(np.concatenate([rows, [0, 31, 32, c.n_rows - 1]]))
    X = np.concatenate([gen_x(2, int(r), 1, 28) for r in rows])
    o = oracle.run(m, X)
    np.testing.assert_array_equal(lab[rows], o["label"])
    np.testing.assert_array_equal(pr[rows], o["proba"])


@pytest.mark.parametrize("n_trees", [40, 150, 270, 300])
def test_chunk_counts_cluster_and_partial_paths(n_trees):
    """2..8 chunks -> one cluster launch with the DSMEM reduction; >8 chunks ->
    per-chunk partials + combine kernel.  Both must match the oracle bitwise."""
    m = perfect_ensemble(13, n_trees, 8, 28, kind="classification", n_classes=2, calib_rows=1024)
    check(m, gen_x(14, 0, 7001, 28), apply=False)


def test_many_deep_chunks_regression():
    m = perfect_ensemble(15, 150, 10, 20, kind="regression", lr=0.01, calib_rows=2048)
    check(m, gen_x(16, 0, 3001, 20), apply=False)


@pytest.mark.parametrize("hybrid", ["1", "0"])
def test_c4_shaped_deep_trees(hybrid, monkeypatch):
    """Depth-12, 8-class trees (164 KB each) exceed shared memory: hybrid mode
    (top levels in shared memory, deep levels + leaves in global) or
    global-tree mode (every CTA walks every tree from global memory)."""
    monkeypatch.setenv("BRIDGER_HYBRID", hybrid)
    # tree-streamed mode is the default for global-tree models (tested below);
    # keep the older global-tree walker reachable and exact
    monkeypatch.setenv("BRIDGER_STREAM", "0")
    c, m = make_config("C4", n_trees=40)
    g, _ = check(m, gen_x(4, 0, 4001, 64))
    assert g.layout()["format"] == ("hybrid" if hybrid == "1" else "heap")  # hybrid is opt-in
    assert g.layout()["global_trees"] == (hybrid == "0")


def test_mixed_depth_forest():
    m = perfect_ensemble(17, 60, 9, 11, kind="classification", n_classes=3, calib_rows=2048)
    m = prune_ensemble(m, 17, p=0.3, with_missing=False)
    check(m, gen_x(18, 0, 5000, 11))


@pytest.mark.parametrize("coded", ["1", "0"])
def test_coded_and_fp32_node_formats(coded, monkeypatch):
    """Threshold-bin codes (§8(f2)) vs plain fp32 nodes: both bit-exact against
    the oracle, including NaN / inf / -0 / subnormal inputs and missing_left."""
    monkeypatch.setenv("BRIDGER_CODES", coded)
    m = perfect_ensemble(27, 90, 8, 21, kind="classification", n_classes=3, calib_rows=2048)
    m = prune_ensemble(m, 27, p=0.1, with_missing=True)
    X = inject_specials(gen_x(28, 0, 6007, 21), 28, rate=0.03)
    X[::97, 3] = m.threshold[m.feature == 3][0]          # exact ties with a threshold
    g, _ = check(m, X)
    assert g.layout()["coded"] == (coded == "1")
    c, m2 = make_config("C3", n_trees=60)
    g2, _ = check(m2, gen_x(3, 0, 4001, 90))
    assert g2.layout()["coded"] == (coded == "1")


@pytest.mark.parametrize("F", [1, 2, 6, 28, 40])
def test_coded_format_feature_widths(F, monkeypatch):
    """Threshold-bin codes at every vector width of the binning kernel (F % 4 =
    0, 2, odd), F = 1, an odd padding feature, ragged row tails; ties placed on
    thresholds, specials injected; bit-exact against the oracle."""
    monkeypatch.setenv("BRIDGER_CODES", "1")
    m = perfect_ensemble(40 + F, 37, 7, F, kind="classification", n_classes=2, calib_rows=2048)
    m = prune_ensemble(m, 40 + F, p=0.05, with_missing=(F % 2 == 0))
    X = inject_specials(gen_x(41 + F, 0, 3001, F), 41 + F, rate=0.02)
    X[::61, 0] = m.threshold[m.feature == 0][0]
    g, _ = check(m, X)
    assert g.layout()["coded"]


@pytest.mark.parametrize("binv", ["coop", "fg", "bucket", "E"])
@pytest.mark.parametrize("F", [7, 28, 90])
def test_coded_binning_variants(binv, F, monkeypatch):
    """The cooperative (CTA-shared block), feature-group (tables per CTA,
    direct loads), bucketed (affine bucket map + short window search) and
    bucket-entry (one 16-byte entry per bucket, TMA-staged row tiles; "E"
    makes it an error if that kernel cannot run) binning kernels produce the
    same codes: bit-exact end to end, with NaN, +-inf, -0 and subnormal
    inputs.  F = 7, 28, 90 cover the 4-, 1- and 2-row super-row views of the
    entry kernel's tensor map, 2011 rows its directly-read tail rows."""
    monkeypatch.setenv("BRIDGER_CODES", "1")
    monkeypatch.setenv("BRIDGER_BIN", binv)
    m = perfect_ensemble(60 + F, 31, 7, F, kind="regression", lr=0.1, calib_rows=2048)
    m = prune_ensemble(m, 60 + F, p=0.05, with_missing=True)
    X = inject_specials(gen_x(61 + F, 0, 2011, F), 61 + F, rate=0.02)
    g, _ = check(m, X)
    assert g.layout()["coded"]


@pytest.mark.parametrize("nbuf", ["2", "3"])
def test_bucketed_binning_many_blocks_per_cta(nbuf, monkeypatch):
    """The all-features bucketed kernel with 10+ row blocks per CTA (every
    staging buffer reused several times: the mbarrier phases of a 2- and a
    3-buffer ring) and a ragged last block filled by hand; C3-shaped, 50,021
    rows, bitwise."""
    monkeypatch.setenv("BRIDGER_CODES", "1")
    monkeypatch.setenv("BRIDGER_BIN", "b")
    monkeypatch.setenv("BRIDGER_BIN_NBUF", nbuf)
    c, m = make_config("C3", n_trees=60)
    X = inject_specials(gen_x(3, 0, 50021, 90), 33, rate=0.01)
    g, _ = check(m, X, apply=False)
    assert g.layout()["coded"]


@pytest.mark.parametrize("F,n", [(7, 129), (7, 131), (90, 130), (28, 160), (90, 4099)])
def test_entry_binning_small_and_ragged(F, n, monkeypatch):
    """Bucket-entry binning (BRIDGER_BIN=E: an error unless that kernel runs)
    at the smallest row counts it takes (>= 128) and ragged sizes: the last
    32-row block partly out of the tensor map (TMA zero fill), rows past the
    last whole R-row super-row read directly (F = 7: R = 4, F = 90: R = 2),
    and a multi-block input; labels, scores and raw sums bitwise."""
    monkeypatch.setenv("BRIDGER_CODES", "1")
    monkeypatch.setenv("BRIDGER_BIN", "E")
    m = perfect_ensemble(70 + F, 23, 6, F, kind="classification", n_classes=3, calib_rows=2048)
    X = inject_specials(gen_x(71 + F, 0, n, F), 71 + F, rate=0.02)
    g, _ = check(m, X)
    assert g.layout()["coded"]


@pytest.mark.parametrize("F,binv", [(4, None), (4, "g"), (5, None), (6, None)])
def test_coded_wide_code_range(F, binv, monkeypatch):
    """Up to 65534 distinct thresholds per feature (16-bit code index, missing
    flag in bit 0): ~164K / F random distinct thresholds per feature ->
    2^16-slot search trees, binned with their top 14 levels in shared memory
    and the rest from global memory -- feature pairs with TMA-staged row
    tiles (F = 4, 5, 6: 1-, 4- and 2-row super-rows) or with direct loads
    (BRIDGER_BIN=g); NaN / missing-left routing included."""
    monkeypatch.setenv("BRIDGER_CODES", "1")
    if binv:
        monkeypatch.setenv("BRIDGER_BIN", binv)
    m = perfect_ensemble(80, 40, 12, F, kind="regression", lr=0.1, calib_rows=512)
    rng = np.random.default_rng(81)
    th = m.threshold.copy()
    internal = m.left != -1
    th[internal] = rng.standard_normal(int(internal.sum())).astype(np.float32)
    ml = (rng.random(len(th)) < 0.3).astype(np.uint8)
    m = ModelDesc(**{**m.__dict__, "threshold": th, "missing_left": ml})
    X = inject_specials(gen_x(82, 0, 3001, F), 82, rate=0.02)
    X[::53, 1] = th[internal][m.feature[internal] == 1][:57].repeat(1)[: len(X[::53])]
    g, _ = check(m, X, apply=False)
    assert g.layout()["coded"]


@pytest.mark.parametrize("binv", [None, "g"])
def test_c5_shard_coded(binv, monkeypatch):
    """C5-shaped tree shard (1250 trees would take minutes in the oracle: 120
    trees of depth 10 over 200 features) in threshold-bin codes with
    feature-group bucketed binning (6K+ thresholds per feature at full size):
    the TMA-staged kernel (default) and the direct-load one (BRIDGER_BIN=g)."""
    monkeypatch.setenv("BRIDGER_CODES", "1")
    if binv:
        monkeypatch.setenv("BRIDGER_BIN", binv)
    c, m = make_config("C5", n_trees=120)
    g, _ = check(m, gen_x(5, 0, 3001, 200), apply=False)


@pytest.mark.parametrize("F", [202, 199])
def test_wide_feature_group_binning_unaligned_rows(F, monkeypatch):
    """Feature-group bucketed tables with TMA row tiles when rows are not
    16-byte aligned (F = 202: 2-row super-rows, F = 199: 4-row), boxes
    starting at the aligned column below each group; NaN / inf / -0 inputs
    and a ragged tail; raw sums bitwise."""
    monkeypatch.setenv("BRIDGER_CODES", "1")
    m = perfect_ensemble(120 + F, 60, 10, F, kind="regression", lr=0.01, calib_rows=2048)
    X = inject_specials(gen_x(121 + F, 0, 2003, F), 121 + F, rate=0.02)
    check(m, X, apply=False)


@pytest.mark.parametrize("pret", ["1", "0"])
def test_pretransposed_input_mode(pret, monkeypatch):
    """Wide input, many chunks: X transposed once into feature-major blocks
    (bulk-copied by every chunk CTA) vs per-chunk transpose -- both exact."""
    monkeypatch.setenv("BRIDGER_PRET", pret)
    c, m = make_config("C5", n_trees=60)
    g, _ = check(m, gen_x(5, 0, 5003, 200), apply=True)
    assert g.layout()["format"] == ("heap_pretransposed" if pret == "1" else "heap")


def test_split_node_format(monkeypatch):
    """Split node arrays (fp32 thresholds + 1-byte features, bit 7 = missing)."""
    monkeypatch.setenv("BRIDGER_SPLIT", "1")
    m = perfect_ensemble(29, 90, 8, 21, kind="classification", n_classes=3, calib_rows=2048)
    m = prune_ensemble(m, 29, p=0.1, with_missing=True)
    X = inject_specials(gen_x(30, 0, 6007, 21), 30, rate=0.03)
    check(m, X)
    c, m2 = make_config("C2", n_trees=100)
    check(m2, gen_x(2, 0, 9001, 28), apply=False)


@pytest.mark.parametrize("split", ["1", "0"])
@pytest.mark.parametrize("n_rows,n_trees", [(77, 6), (513, 7), (148 * 512 + 333, 6)])
def test_tree_streamed_c4_shape(n_rows, n_trees, split, monkeypatch):
    # C4-shaped trees (depth 12, 8 classes: 164 KB per tree) exceed shared
    # memory: tree-streamed mode (row tiles resident, node records streamed),
    # split (5-byte, two trees per ring slot; odd tree counts leave a one-tree
    # slot) or 8-byte node records
    monkeypatch.setenv("BRIDGER_STREAM_SPLIT", split)
    c, m = make_config("C4", n_trees=n_trees)
    g = B.Model(m)
    assert g.layout()["format"] == "stream"
    check(m, gen_x(4, 0, n_rows, 64), apply=n_rows < 1000)


@pytest.mark.parametrize("n_rows,n_trees,ml", [(77, 6, False), (513, 7, True), (300, 5, False), (148 * 512 + 333, 6, False)])
def test_tree_streamed_codes(n_rows, n_trees, ml, monkeypatch):
    """Tree-streamed mode in threshold-bin codes (C4-shaped: depth 12, 8
    classes): u16 code blocks as the row tile, 4-byte node words streamed two
    trees per slot; odd tree counts, tail tiles, specials and missing-left."""
    monkeypatch.setenv("BRIDGER_CODES", "1")
    c, m = make_config("C4", n_trees=n_trees)
    if ml:
        m = prune_ensemble(m, 97, p=0.0005, with_missing=True)
    g = B.Model(m)
    assert g.layout()["format"] == "stream_codes"
    X = gen_x(4, 0, n_rows, 64)
    if ml:
        X = inject_specials(X, 98, rate=0.02)
    check(m, X, apply=n_rows < 1000)


def test_tree_streamed_codes_many_classes(monkeypatch):
    """Streamed codes with K = 12 (leaf vectors gathered by 4-byte cp.async
    into element-major landing slots, KT = 16 != K) and an odd feature count."""
    monkeypatch.setenv("BRIDGER_CODES", "1")
    m = perfect_ensemble(120, 5, 12, 21, kind="classification", n_classes=12, calib_rows=2048)
    g = B.Model(m)
    assert g.layout()["format"] == "stream_codes"
    check(m, inject_specials(gen_x(121, 0, 1500, 21), 121, rate=0.01))


def test_tree_streamed_codes_f64_tier(monkeypatch):
    """Streamed codes with fp64 accumulation (a subnormal leaf value forces the
    F64 tier, reading c9): scores within the tolerance, labels exact."""
    monkeypatch.setenv("BRIDGER_CODES", "1")
    c, m = make_config("C4", n_trees=5)
    v = m.value.copy()
    v[np.nonzero(m.left == -1)[0][0] * m.n_outputs] = np.float32(1.4e-45)
    m = ModelDesc(**{**m.__dict__, "value": v})
    assert B.analyze_exactness(m)[1] == "F64"
    g = B.Model(m)
    assert g.layout()["format"] == "stream_codes"
    check(m, gen_x(4, 0, 1200, 64), exact=False, apply=False)


@pytest.mark.parametrize("ml", [False, True])
def test_tree_streamed_pruned_missing_mixed_depth(ml):
    m = perfect_ensemble(95, 10, 12, 64, kind="classification", n_classes=8, calib_rows=2048)
    m = prune_ensemble(m, 95, p=0.003, with_missing=ml)  # heavier pruning selects the sparse layout
    g = B.Model(m)
    assert g.layout()["format"] == "stream"
    check(m, inject_specials(gen_x(96, 0, 2001, 64), 96, rate=0.02))


@pytest.mark.parametrize("spread", ["clustered", "wide", "single", "bunched"])
def test_bucketed_binning_threshold_layouts(spread, monkeypatch):
    """Bucketed binning on threshold sets that stress the bucket map: many
    thresholds packed into a tiny range (large per-bucket counts: the window
    search, or the fallback to the Eytzinger kernels when a bucket exceeds
    15), thresholds spread over 1e-30..1e30, and features with a single
    distinct threshold (zero span); inputs placed exactly on, just below and
    just above every threshold.  Bit-exact against the oracle either way."""
    monkeypatch.setenv("BRIDGER_CODES", "1")
    F = 6
    m = perfect_ensemble(83, 40, 6, F, kind="regression", lr=0.1, calib_rows=1024)
    thr = np.array(m.threshold, np.float32)
    inner = np.asarray(m.left) != -1
    rng = np.random.default_rng(7)
    n_in = int(inner.sum())
    if spread == "clustered":
        vals = np.float32(1.0) + rng.integers(0, 200, n_in).astype(np.float32) * np.float32(2.0 ** -23)
    elif spread == "wide":
        vals = (rng.choice([-1, 1], n_in) * 10.0 ** rng.uniform(-30, 30, n_in)).astype(np.float32)
    elif spread == "bunched":
        # 50 bunches of 8 thresholds 1e-6 apart: 4..15 per bucket, so the
        # entry kernel's overflow window search runs next to its 1-load path
        base = np.repeat(np.arange(50, dtype=np.float32) / np.float32(50), 8)
        vals = (base + np.tile(np.arange(8, dtype=np.float32), 50) * np.float32(1e-6))[rng.integers(0, 400, n_in)]
    else:
        vals = np.full(n_in, 0.25, np.float32)
    thr[inner] = vals
    m.threshold = thr
    u = np.unique(vals)
    base = gen_x(84, 0, 3000, F)
    pick = rng.choice(u, size=base.shape)
    jitter = rng.integers(-1, 2, size=base.shape)
    X = np.where(jitter < 0, np.nextafter(pick, np.float32(-np.inf)),
                 np.where(jitter > 0, np.nextafter(pick, np.float32(np.inf)), pick)).astype(np.float32)
    X[::97, 1] = np.nan
    X[::89, 2] = np.inf
    X[::83, 3] = -np.inf
    X[::79, 4] = -0.0
    for binv in ("bucket", "coop", "e" if spread == "wide" else "E"):
        monkeypatch.setenv("BRIDGER_BIN", binv)
        check(m, X)


@pytest.mark.parametrize("K,ml", [(1, True), (2, True), (2, False), (3, True)])
def test_deep_chunks_speculative_walk_variants(K, ml, monkeypatch):
    """K4d on deep (depth 10, after pruning: mixed-depth, replicated leaves)
    coded trees in >= 2 chunks, every walk variant: child-pair speculation
    with missing-left routing (ML) for K = 1 (single last-level leaf) and K = 2
    (leaf-pair vector), and the non-speculative walk for K = 3 (K != KT);
    NaN / +-inf / -0 / subnormal inputs, a ragged last block; labels, proba,
    scores and raw int64 sums bitwise (E53)."""
    monkeypatch.setenv("BRIDGER_CODES", "1")
    kind = "regression" if K == 1 else "classification"
    m = perfect_ensemble(90 + K, 60, 10, 24, kind=kind, n_classes=K, lr=0.02, calib_rows=2048)
    m = prune_ensemble(m, 90 + K, p=0.05, with_missing=ml)
    X = inject_specials(gen_x(91 + K, 0, 2077, 24), 91 + K, rate=0.02)
    g, _ = check(m, X, apply=False)
    assert g.layout()["format"] == "codes_deep", g.layout()
    raw = g.predict_raw(dev(X)).cpu().numpy()
    want = np.round(np.ldexp(oracle.run(m, X)["acc"], -g.info()["acc_scale_exp"])).astype(np.int64)
    np.testing.assert_array_equal(raw, want)

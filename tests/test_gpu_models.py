"""Real-model and edge-tier parity on the GPU: scikit-learn-trained trees
(unbalanced, mixed depths up to 14, NaN routing), the E63 exactness tier
(int64 exact, oracle within 1e-5; shard/permutation invariance bitwise), many
classes (K > 8 register-array paths), and K = 1 regression through the host
API."""
import numpy as np
import pytest

import oracle
from synth import gen_x, inject_specials, make_config, perfect_ensemble
from synth.trees import ModelDesc
from tests.sk_export import from_sklearn_forest, from_sklearn_gbr
from tests.test_gpu_parity import check, dev

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
import paper_2405_12491_b200 as B  # noqa: E402

sk = pytest.importorskip("sklearn")
from sklearn.ensemble import GradientBoostingRegressor, RandomForestClassifier  # noqa: E402
from sklearn.tree import DecisionTreeClassifier  # noqa: E402


def _data(seed, n, F, k, nan_rate=0.0):
    X = gen_x(seed, 0, n, F)
    z = X @ np.linspace(-1, 1, F).astype(np.float32) + 0.5 * X[:, 0] * X[:, 1]
    y = np.digitize(z, np.quantile(z, np.linspace(0, 1, k + 1)[1:-1]))
    if nan_rate:
        X = inject_specials(X, seed, rate=nan_rate)
        X[np.isinf(X)] = 0
    return X, y, z


@pytest.mark.parametrize("variant", ["traverse", "gemm"])
def test_sklearn_random_forest_unbounded_depth(variant):
    X, y, _ = _data(31, 6000, 12, 5, nan_rate=0.01)
    depth = 14 if variant == "traverse" else 8
    est = RandomForestClassifier(n_estimators=40, max_depth=depth, random_state=0).fit(X, y)
    m = from_sklearn_forest(est, 12, with_missing=True)
    Xt, _, _ = _data(32, 4001, 12, 5, nan_rate=0.01)
    g, o = check(m, Xt, variant=variant, apply=variant == "traverse")
    np.testing.assert_allclose(g.predict_proba(dev(Xt)).cpu().numpy(), est.predict_proba(Xt), atol=1e-6)


def test_sklearn_decision_tree_deep():
    X, y, _ = _data(33, 20000, 6, 3)
    est = DecisionTreeClassifier(max_depth=14, random_state=0).fit(X, y)
    m = from_sklearn_forest(est, 6)
    Xt, _, _ = _data(34, 5000, 6, 3)
    g, _ = check(m, Xt)
    np.testing.assert_array_equal(g.apply(dev(Xt)).cpu().numpy()[:, 0], est.apply(Xt))


def test_sklearn_gbr():
    X, _, z = _data(35, 5000, 7, 2)
    est = GradientBoostingRegressor(n_estimators=80, max_depth=5, random_state=0).fit(X, z)
    m = from_sklearn_gbr(est, 7, X)
    Xt, _, _ = _data(36, 3000, 7, 2)
    g, _ = check(m, Xt)
    np.testing.assert_allclose(g.predict(dev(Xt)).cpu().numpy()[:, 0], est.predict(Xt), rtol=1e-5, atol=1e-6)


def test_e63_tier_exact_and_order_free():
    m = perfect_ensemble(41, 64, 6, 8, kind="regression", lr=1.0)
    v = m.value.copy()
    leaves = np.nonzero(m.left == -1)[0]
    # every value a multiple of 2^-10 (q = -10) with per-tree maxima 2^42:
    # M = 64 * 2^42 * 2^10 = 2^58 -> tier E63 (fp64 sums of such values round)
    v[leaves] = np.round(v[leaves] * 1024) / np.float32(1024)
    v[leaves[::3]] = np.float32(2.0 ** 42) * np.sign(v[leaves[::3]] + 1e-30)
    v[leaves[1]] = np.float32(2.0 ** -10)
    m = ModelDesc(**{**m.__dict__, "value": v.astype(np.float32)})
    q, tier, l2 = B.analyze_exactness(m)
    assert tier == "E63", (tier, l2)
    X = gen_x(42, 0, 3000, 8)
    g = B.Model(m)
    assert g.info()["acc_is_int64"] and g.info()["acc_scale_exp"] == q
    raw = g.predict_raw(dev(X))
    # exact reference: integer sum of the leaf values the oracle's walk reached
    o = oracle.run(m, X)
    offs = m.tree_offsets
    ints = np.round(np.ldexp(m.value.astype(np.float64), -q)).astype(np.int64)
    exact = np.zeros(X.shape[0], np.int64)
    for t in range(m.n_trees):
        exact += ints[offs[t] + o["leaf"][:, t]]
    np.testing.assert_array_equal(raw.cpu().numpy()[:, 0], exact)
    # finalize from the exact sum, same fp64 operations as the definition (c6)
    a = exact.astype(np.float64) * 2.0 ** q
    want = (np.float64(0.5) + np.float64(m.leaf_scale) * a).astype(np.float32)
    np.testing.assert_array_equal(g.predict(dev(X)).cpu().numpy()[:, 0], want)
    # the oracle's fp64 tree-order sum is within its own rounding bound of the exact sum
    bound = m.n_trees * 2.0 ** -52 * np.max(np.abs(m.value)) * m.n_trees
    assert np.max(np.abs(o["acc"][:, 0] - a)) <= bound
    # int64 accumulation is order-free: a permuted ensemble gives identical bits
    perm = np.random.default_rng(1).permutation(m.n_trees)
    assert torch.equal(raw, B.Model(m.subset(perm)).predict_raw(dev(X)))


@pytest.mark.parametrize("K", [9, 16, 33])
def test_many_classes(K):
    m = perfect_ensemble(43, 25, 5, 10, kind="classification", n_classes=K, calib_rows=512)
    check(m, gen_x(44, 0, 2001, 10))


def test_regression_host_api():
    m = perfect_ensemble(45, 30, 6, 12, kind="regression")
    X = gen_x(46, 0, 50001, 12)
    g = B.Model(m)
    out = g.predict_host(X).numpy()
    np.testing.assert_array_equal(out, oracle.run(m, X)["pred"])


def test_sklearn_unbounded_depth_forest_sparse_layout():
    """sklearn's default max_depth=None: deep, unbalanced trees (beyond any
    perfect-heap padding) run in the sparse pointer layout (§8(f3))."""
    X, y, _ = _data(51, 30000, 10, 4, nan_rate=0.005)
    est = RandomForestClassifier(n_estimators=12, max_depth=None, random_state=0).fit(X, y)
    assert max(e.tree_.max_depth for e in est.estimators_) > 14
    m = from_sklearn_forest(est, 10, with_missing=True)
    Xt, _, _ = _data(52, 7001, 10, 4, nan_rate=0.005)
    g, _ = check(m, Xt)
    assert g.layout()["format"] == "sparse"
    np.testing.assert_array_equal(g.apply(dev(Xt)).cpu().numpy(), est.apply(Xt))
    np.testing.assert_allclose(g.predict_proba(dev(Xt)).cpu().numpy(), est.predict_proba(Xt), atol=1e-6)


def test_sparse_layout_forced_matches_heap(monkeypatch):
    m = perfect_ensemble(53, 50, 7, 9, kind="regression", calib_rows=1024)
    X = gen_x(54, 0, 4001, 9)
    a = B.Model(m).predict(dev(X)).cpu().numpy()
    monkeypatch.setenv("BRIDGER_SPARSE", "1")
    g = B.Model(m)
    assert g.layout()["format"] == "sparse"
    np.testing.assert_array_equal(g.predict(dev(X)).cpu().numpy(), a)
    check(m, X)


@pytest.mark.parametrize("variant", ["traverse", "gemm", "gemm_staged"])
def test_multiclass_gbdt_softmax(variant):
    # reading c15: K scalar-leaf trees per round, SUM aggregation, softmax proba
    from synth import multiclass_gbdt
    m = multiclass_gbdt(81, 30, 6, 14, 5)
    X = inject_specials(gen_x(82, 0, 6001, 14), 82, rate=0.01)
    g, o = check(m, X, variant=variant, apply=variant == "traverse")
    assert g.info()["exact_tier"] == "E53"


def test_sklearn_gradient_boosting_classifier_multiclass():
    from sklearn.ensemble import GradientBoostingClassifier
    from tests.sk_export import from_sklearn_gbc_multiclass
    X, y, _ = _data(37, 5000, 8, 4)
    est = GradientBoostingClassifier(n_estimators=40, max_depth=4, learning_rate=0.2, random_state=0).fit(X, y)
    m = from_sklearn_gbc_multiclass(est, 8, X)
    Xt, _, _ = _data(38, 3000, 8, 4)
    g, _ = check(m, Xt, exact=False)
    np.testing.assert_array_equal(g.apply(dev(Xt)).cpu().numpy(), est.apply(Xt).reshape(len(Xt), -1))
    np.testing.assert_allclose(g.predict_proba(dev(Xt)).cpu().numpy(), est.predict_proba(Xt), rtol=1e-5, atol=1e-6)


@pytest.mark.parametrize("name", ["xgboost_binary_logistic.json", "xgboost_multiclass_softprob.json",
                                  "lightgbm_binary_dump.json"])
def test_imported_formats_on_gpu(name):
    from paper_2405_12491_b200 import importers as I
    from tests.helpers import load_golden, parse_x
    g = load_golden(name)
    m = I.from_lightgbm_json(g["model"]) if name.startswith("lightgbm") else I.from_xgboost_json(g["model"])
    X = parse_x(g["X"])
    # the hand rows, then a larger seeded batch with specials through the same model
    Xb = np.concatenate([X, inject_specials(gen_x(93, 0, 3000, m.n_features), 93, rate=0.05)])
    check(m, Xb, exact=False)


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two GPUs in one process")
def test_two_devices_one_process():
    """the >48 KB shared-memory opt-in is per device; models on two
    GPUs of one process (loaded and run alternately) must both launch."""
    _, m = make_config("C3", n_trees=60)
    X = gen_x(3, 0, 4099, 90)
    o = oracle.run(m, X)
    for dev_i in (0, 1, 0, 1):
        g = B.Model(m, device=dev_i)
        xd = torch.from_numpy(X).to(f"cuda:{dev_i}")
        with torch.cuda.device(dev_i):
            got = g.predict(xd).cpu().numpy()
        np.testing.assert_array_equal(got, o["pred"])


def test_predict_on_caller_stream():
    """Kernels are enqueued on the caller's current stream (the boundary's
    stream argument, filled by the binding from torch's current stream): a
    predict issued on a side stream behind a long kernel on that stream sees
    the input that kernel wrote, and the default stream is not used."""
    c, m = make_config("C2", n_trees=20)
    g = B.Model(m)
    X = gen_x(2, 0, 4096, 28)
    want = oracle.run(m, X)["label"]
    Xd = torch.zeros((4096, 28), device="cuda")
    src = torch.from_numpy(X).cuda()
    big = torch.empty(64 << 20, device="cuda")
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        big.fill_(1.0)          # keeps the side stream busy
        Xd.copy_(src)           # the input appears only after it
        lab = g.predict(Xd)
    s.synchronize()
    np.testing.assert_array_equal(lab.cpu().numpy(), want)


@pytest.mark.parametrize("name,trees", [("C1", None), ("C2", 20), ("C3", 240), ("C5", 60)])
def test_predict_captured_in_cuda_graph(name, trees):
    """A predict call captured into a CUDA graph (serving: one graph launch per
    batch instead of the binding + host dispatch) and replayed on new input
    contents gives the oracle's answers: binning, the walk kernels (K4, K4d
    with programmatic dependent launch), stream-ordered scratch and finalize
    are all capturable."""
    cfg, m = make_config(name, n_trees=trees)
    n = 150 if name == "C1" else 3000
    g = B.Model(m)
    if name == "C3":
        assert g.layout()["format"] == "codes_deep"  # K4d (PDL launch) inside the graph
    Xs = [gen_x(cfg.seed + i, 0, n, cfg.n_features) for i in range(3)]
    Xd = torch.from_numpy(Xs[0]).cuda()
    classif = cfg.kind == "classification"
    out = torch.empty(n, dtype=torch.int32, device="cuda") if classif else torch.empty((n, cfg.n_classes), device="cuda")
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        g.predict(Xd, out=out)  # warm-up (attributes, pools) outside the capture
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        g.predict(Xd, out=out)
    for X in Xs[1:] + Xs[:1]:
        Xd.copy_(torch.from_numpy(X))
        graph.replay()
        torch.cuda.synchronize()
        o = oracle.run(m, X)
        if classif:
            np.testing.assert_array_equal(out.cpu().numpy(), o["label"])
        else:
            np.testing.assert_array_equal(out.cpu().numpy(), o["pred"].astype(np.float32).reshape(out.shape))

"""Linear models on the GPU (bridger_linear_*) against the
oracle (oracle_linear_run): fp64 scores bit-identical (same operation order,
no FMA), labels exact, sigmoid/softmax probabilities within 1e-5 (c10); the
StandardScaler transform in fp32 (c16).  Sizes span many 32-row blocks,
persistent-CTA strides and a ragged tail; wide inputs (one warp per CTA) and
K = 64 outputs."""
from types import SimpleNamespace

import numpy as np
import pytest

import oracle
from synth import gen_x, inject_specials
from tests.helpers import load_golden, parse_x

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
import paper_2405_12491_b200 as B  # noqa: E402
from paper_2405_12491_b200 import importers as I  # noqa: E402


def dev(X):
    return torch.from_numpy(np.ascontiguousarray(X)).cuda()


def _rand_linear(seed, F, K, task, post, scaler=False):
    rng = np.random.default_rng(seed)
    return SimpleNamespace(n_features=F, n_outputs=K, coef=rng.normal(size=(K, F)) * 0.3,
                           intercept=rng.normal(size=K) * 0.1,
                           mean=rng.normal(size=F) if scaler else None,
                           scale=rng.uniform(0.5, 2.0, size=F) if scaler else None, task=task, post=post)


def check_linear(m, X):
    g = B.LinearModel(m)
    o = oracle.run_linear(m, X)
    Xd = dev(X)
    s = g.decision_function(Xd).cpu().numpy()
    np.testing.assert_array_equal(s, o["s"])
    if int(m.task) == 1:
        np.testing.assert_array_equal(g.predict(Xd).cpu().numpy(), o["label"])
        np.testing.assert_allclose(g.predict_proba(Xd).cpu().numpy(), o["proba"], rtol=1e-5, atol=1e-7)
    else:
        np.testing.assert_array_equal(g.predict(Xd).cpu().numpy(), o["pred"])
    return g, o


@pytest.mark.parametrize("case", ["binary", "binary_scaled", "multiclass"])
def test_linear_hand_golden_on_gpu(case):
    g = load_golden("linear_models_hand.json")
    c = g[case]
    m = SimpleNamespace(n_features=2, n_outputs=len(c["coef"]), coef=np.asarray(c["coef"]),
                        intercept=np.asarray(c["intercept"]), mean=c.get("mean"), scale=c.get("scale"),
                        task=1, post=2 if case == "multiclass" else 1)
    check_linear(m, parse_x(g["X"]))


@pytest.mark.parametrize("F,K,task,post,scaler,n", [
    (28, 1, 1, 1, False, 100003), (28, 1, 1, 1, True, 4099), (90, 5, 1, 2, True, 20011),
    (90, 1, 0, 0, False, 50001), (13, 3, 0, 0, True, 777), (500, 4, 1, 2, False, 3001),
    (17, 64, 1, 2, False, 2001), (7, 10, 1, 0, False, 33)])
def test_linear_random_models(F, K, task, post, scaler, n):
    m = _rand_linear(F * 100 + K, F, K, task, post, scaler)
    X = gen_x(F + K, 0, n, F)
    check_linear(m, X)


def test_linear_specials_and_empty():
    m = _rand_linear(5, 11, 3, 1, 2, scaler=True)
    X = inject_specials(gen_x(6, 0, 2000, 11), 6, rate=0.01)
    X[np.isnan(X)] = 0.0  # NaN inputs give NaN scores (well defined, but argmax of NaN is not compared)
    check_linear(m, X)
    g = B.LinearModel(m)
    assert g.predict(torch.empty((0, 11), device="cuda")).shape[0] == 0


@pytest.mark.parametrize("F,offset", [(28, 0), (28, 1), (28, 2), (90, 0), (90, 1), (64, 3)])
def test_linear_copy_widths_and_misaligned_input(F, offset):
    """The staging copies are 16-, 8- or 4-byte vectors, the widest that divides
    F and the alignment of X: a view starting `offset` floats into its buffer
    forces the narrower copies (F = 28: 16 B aligned -> 8 B -> 4 B)."""
    m = _rand_linear(F + offset, F, 3, 1, 2, scaler=offset % 2 == 1)
    n = 4133
    X = gen_x(F * 7 + offset, 0, n, F)
    buf = torch.zeros(n * F + offset, dtype=torch.float32, device="cuda")
    Xd = buf[offset:].view(n, F)
    Xd.copy_(dev(X))
    g = B.LinearModel(m)
    o = oracle.run_linear(m, X)
    np.testing.assert_array_equal(g.decision_function(Xd).cpu().numpy(), o["s"])
    np.testing.assert_array_equal(g.predict(Xd).cpu().numpy(), o["label"])


def test_linear_c3_shape_full_size_sampled():
    """At the size tools/bench_linear.py times (10M x 90, K = 1 regression), in
    its launch configuration: sampled rows against the oracle, bitwise."""
    F, n = 90, 10_000_000
    m = _rand_linear(99, F, 1, 0, 0)
    from synth import gen_x_torch
    Xd = gen_x_torch(11, 0, n, F, device="cuda")
    out = B.LinearModel(m).predict(Xd).cpu().numpy()
    rows = np.unique(np.concatenate([np.arange(64), np.random.default_rng(3).integers(0, n, 2000), np.arange(n - 64, n)]))
    Xs = np.stack([gen_x(11, int(r), 1, F)[0] for r in rows])  # counter-based: any row on its own
    np.testing.assert_array_equal(out[rows], oracle.run_linear(m, Xs)["pred"])


sk = pytest.importorskip("sklearn")


def test_sklearn_pipeline_logistic_regression():
    from sklearn.linear_model import LogisticRegression
    from sklearn.pipeline import make_pipeline
    from sklearn.preprocessing import StandardScaler
    X = gen_x(71, 0, 4000, 12) * np.float32(2.0) + np.float32(0.5)
    z = X @ np.linspace(-1, 1, 12).astype(np.float32)
    y = np.digitize(z, np.quantile(z, [0.3, 0.6]))
    pipe = make_pipeline(StandardScaler(), LogisticRegression(max_iter=400)).fit(X, y)
    m = I.from_sklearn_linear(pipe)
    Xt = gen_x(72, 0, 3000, 12) * np.float32(2.0) + np.float32(0.5)
    g, o = check_linear(m, Xt)
    # sklearn itself (fp32 model, sgemm order): probabilities within 1e-5
    np.testing.assert_allclose(g.predict_proba(dev(Xt)).cpu().numpy(), pipe.predict_proba(Xt), rtol=1e-4, atol=1e-5)

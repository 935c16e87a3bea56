"""Randomised shapes through the production path (AUTO variant, every layout
and binning kernel the lowering picks for them) against the oracle: feature
counts 1..300 (odd and even, 1-, 2- and 4-row TMA super-rows), 1..400 trees,
depths 1..12, K = 1, 2, 3, 8, pruned trees with missing-left routing, row
counts from 1 to ~70K (ragged 32-row blocks and tiles), specials in the input,
forced threshold-bin codes on half the cases.  The seed list is fixed, so the
test is deterministic; each case is small enough for the oracle.  Bar: labels
and leaf indices bitwise; scores and raw sums bitwise in tier E53, else 1e-5
(BASELINE.json north_star)."""
import numpy as np
import pytest

import oracle
from synth import gen_x, inject_specials, perfect_ensemble, prune_ensemble

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
import paper_2405_12491_b200 as B  # noqa: E402


def _case(seed):
    r = np.random.default_rng(1000 + seed)
    F = int(r.choice([1, 2, 3, 5, 7, 21, 28, 64, 90, 127, 200, 300]))
    D = int(r.integers(1, 13))
    T = int(r.integers(1, 400 if D <= 8 else 60))
    K = int(r.choice([1, 2, 3, 8]))
    kind = "regression" if K == 1 and r.random() < 0.6 else "classification"
    if kind == "classification" and K == 1:
        K = 2
    n = int(r.choice([1, 31, 33, 129, 1000, 4099, int(r.integers(5000, 70000))]))
    prune = r.random() < 0.5
    codes = r.random() < 0.5
    return F, D, T, K, kind, n, prune, codes


@pytest.mark.parametrize("seed", list(range(64)))
def test_fuzz_shapes(seed, monkeypatch):
    F, D, T, K, kind, n, prune, codes = _case(seed)
    # the oracle's cost: keep every case to a few seconds
    while n * T * D > 60_000_000 and n > 1000:
        n //= 2
    if codes:
        monkeypatch.setenv("BRIDGER_CODES", "1")
    m = perfect_ensemble(2000 + seed, T, D, F, kind=kind, n_classes=K if kind == "classification" else 1,
                         lr=0.05, calib_rows=1024)
    if prune:
        m = prune_ensemble(m, 3000 + seed, p=0.08, with_missing=True)
    X = inject_specials(gen_x(4000 + seed, 0, n, F), 5000 + seed, rate=0.01)
    g = B.Model(m)
    o = oracle.run(m, X)
    Xd = torch.from_numpy(np.ascontiguousarray(X)).cuda()
    info = g.info()
    exact = info["exact_tier"] == "E53"
    tag = f"F={F} D={D} T={T} K={K} {kind} n={n} prune={prune} codes={codes} layout={g.layout()['format']}"
    if m.task == 1:
        np.testing.assert_array_equal(g.predict(Xd).cpu().numpy(), o["label"], err_msg=tag)
    else:
        got = g.predict(Xd).cpu().numpy()
        if exact:
            np.testing.assert_array_equal(got, o["pred"], err_msg=tag)
        else:
            np.testing.assert_allclose(got, o["pred"], rtol=1e-5, atol=1e-6, err_msg=tag)
    np.testing.assert_array_equal(g.apply(Xd).cpu().numpy(), o["leaf"], err_msg=tag)
    if m.task == 1:
        pr = g.predict_proba(Xd).cpu().numpy()
        if exact and m.post == 0:
            np.testing.assert_array_equal(pr, o["proba"], err_msg=tag)
        else:
            np.testing.assert_allclose(pr, o["proba"], rtol=1e-5, atol=1e-7, err_msg=tag)
    # the end-to-end host-buffer API (chunked H2D / compute / D2H pipeline)
    host = g.predict_host(X).numpy()
    np.testing.assert_array_equal(host, g.predict(Xd).cpu().numpy(), err_msg=tag)
    raw = g.predict_raw(Xd).cpu().numpy()
    a = raw.astype(np.float64) * 2.0 ** info["acc_scale_exp"] if info["acc_is_int64"] else raw
    if exact:
        np.testing.assert_array_equal(a, o["acc"], err_msg=tag)
    else:
        np.testing.assert_allclose(a, o["acc"], rtol=1e-9, atol=1e-12, err_msg=tag)


@pytest.mark.parametrize("variant", ["gemm", "gemm_staged", "gemm_sparse"])
@pytest.mark.parametrize("seed", list(range(12)))
def test_fuzz_gemm_variants(seed, variant):
    """The paper's GEMM form (fused K5, staged K1->K2->K3, 2:4-sparse K2s) on
    randomised shapes of depth <= 8 (the path matrix's range) vs the oracle."""
    F, D, T, K, kind, n, prune, _ = _case(100 + seed)
    D = min(D, 8)
    T = min(T, 120)
    n = min(n, 6000)
    m = perfect_ensemble(6000 + seed, T, D, F, kind=kind, n_classes=K if kind == "classification" else 1,
                         lr=0.05, calib_rows=1024)
    if prune:
        m = prune_ensemble(m, 7000 + seed, p=0.08, with_missing=True)
    X = inject_specials(gen_x(8000 + seed, 0, n, F), 9000 + seed, rate=0.01)
    g = B.Model(m, variant=variant)
    o = oracle.run(m, X)
    Xd = torch.from_numpy(np.ascontiguousarray(X)).cuda()
    tag = f"{variant} F={F} D={D} T={T} K={K} {kind} n={n} prune={prune}"
    exact = g.info()["exact_tier"] == "E53"
    if m.task == 1:
        np.testing.assert_array_equal(g.predict(Xd).cpu().numpy(), o["label"], err_msg=tag)
    elif exact:
        np.testing.assert_array_equal(g.predict(Xd).cpu().numpy(), o["pred"], err_msg=tag)
    else:
        np.testing.assert_allclose(g.predict(Xd).cpu().numpy(), o["pred"], rtol=1e-5, atol=1e-6, err_msg=tag)

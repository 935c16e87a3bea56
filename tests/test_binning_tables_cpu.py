"""CPU pins of the threshold-bin code tables (step a1 in coded form,
PAPER.md:502 "data type rewriting"; DESIGN.md §6 bucketed / bucket-entry
binning).  The definition: code(x) = #{distinct thresholds of feature f that
are < x} (so x <= U_f[j] <=> code(x) <= j), 0xFFFF for NaN.  The library's
host emulation of both bucket tables (bridger_bin_codes_host: the same fp32
bucket map, cum table / 16-byte entries and 15-wide window the kernels use)
must equal that definition computed here with numpy's searchsorted on the
distinct thresholds read from the original node arrays -- on inputs that sit
exactly on, one ulp below and one ulp above every threshold, specials, and
threshold layouts that stress the map (dense bunches, a single threshold,
values spanning 1e-30..1e30, where the tables are not built)."""
import numpy as np
import pytest

import paper_2405_12491_b200 as B
from synth import gen_x, inject_specials, make_config, perfect_ensemble

pytestmark = pytest.mark.filterwarnings("ignore::RuntimeWarning")


def definition_codes(m, X):
    feat, thr, left = np.asarray(m.feature), np.asarray(m.threshold, np.float32), np.asarray(m.left)
    out = np.empty(X.shape, np.uint16)
    for f in range(X.shape[1]):
        u = np.unique(thr[(left != -1) & (feat == f)])
        c = np.searchsorted(u, X[:, f], side="left").astype(np.int64)
        c[np.isnan(X[:, f])] = 0xFFFF
        out[:, f] = c
    return out


def probe_inputs(m, seed, n, F):
    """Random rows, then rows placed on / one ulp around thresholds, specials."""
    rng = np.random.default_rng(seed)
    X = gen_x(seed, 0, n, F)
    thr = np.asarray(m.threshold, np.float32)[np.asarray(m.left) != -1]
    pick = rng.choice(thr, size=(n, F))
    jit = rng.integers(-1, 2, size=(n, F))
    near = np.where(jit < 0, np.nextafter(pick, np.float32(-np.inf)),
                    np.where(jit > 0, np.nextafter(pick, np.float32(np.inf)), pick)).astype(np.float32)
    X = np.concatenate([X, near])
    return inject_specials(X, seed + 1, rate=0.02)


def check_tables(m, X, want_built=True):
    want = definition_codes(m, X)
    for method in ("bucket", "entry"):
        codes, nb = B.bin_codes_host(m, X, method)
        if nb == 0:
            assert not want_built or method == "bucket", f"{method} table not built"
            continue
        mism = np.argwhere(codes != want)
        assert mism.size == 0, (method, nb, mism[:5], X[tuple(mism[0])], codes[tuple(mism[0])], want[tuple(mism[0])])


@pytest.mark.parametrize("name", ["C2", "C3"])
def test_config_tables(name):
    """C2 (RF, ~900 thresholds per feature) and C3 (GBDT, ~350): both tables
    built and equal to the definition."""
    cfg, m = make_config(name)
    X = probe_inputs(m, 11, 4000, cfg.n_features)
    check_tables(m, X)


@pytest.mark.parametrize("spread", ["bunched", "clustered", "single", "wide"])
def test_threshold_layouts(spread):
    """Bunches of 8 thresholds 1e-6 apart (4..15 per bucket: the entry table's
    window path), 200 thresholds within 200 ulps, one threshold per feature
    (zero span), and 1e-30..1e30 (an overfull bucket: no table, nb == 0)."""
    F = 6
    m = perfect_ensemble(83, 40, 6, F, kind="regression", lr=0.1, calib_rows=1024)
    thr = np.array(m.threshold, np.float32)
    inner = np.asarray(m.left) != -1
    rng = np.random.default_rng(7)
    n_in = int(inner.sum())
    if spread == "bunched":
        base = np.repeat(np.arange(50, dtype=np.float32) / np.float32(50), 8)
        vals = (base + np.tile(np.arange(8, dtype=np.float32), 50) * np.float32(1e-6))[rng.integers(0, 400, n_in)]
    elif spread == "clustered":
        vals = np.float32(1.0) + rng.integers(0, 200, n_in).astype(np.float32) * np.float32(2.0 ** -23)
    elif spread == "single":
        vals = np.full(n_in, 0.25, np.float32)
    else:
        vals = (rng.choice([-1, 1], n_in) * 10.0 ** rng.uniform(-30, 30, n_in)).astype(np.float32)
    thr[inner] = vals
    m.threshold = thr
    X = probe_inputs(m, 12, 3000, F)
    X[::89, 2] = np.inf
    X[::83, 3] = -np.inf
    X[::79, 4] = -0.0
    if spread == "wide":
        for method in ("bucket", "entry"):
            codes, nb = B.bin_codes_host(m, X, method)
            assert nb == 0 and codes is None
    else:
        check_tables(m, X)
        if spread == "bunched":  # the entry table really has overfull (window) buckets here
            _, nb = B.bin_codes_host(m, X, "entry")
            assert nb > 0


def test_rejects_uncoded_and_bad_args():
    """A single shallow tree stays in the fp32 node format: E_UNSUPPORTED."""
    c, m = make_config("C1")
    X = np.zeros((4, 4), np.float32)
    with pytest.raises(B.BridgerError):
        B.bin_codes_host(m, X, "entry")
    with pytest.raises(KeyError):
        B.bin_codes_host(m, X, "nope")

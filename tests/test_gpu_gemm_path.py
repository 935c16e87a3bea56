"""GEMM-form path (steps a1..a4 as K1 gather-compare, K2 tcgen05 int8 path
contraction, K3 leaf gather/reduce) against definitions the mathematics fixes:

* K1 decisions P[t][r][i] == [x[r, A_t[i]] <= B_t[i]] (NaN -> missing_left),
  computed on the CPU from the library's own padded heap arrays, bitwise;
* K2 S == P . C_D as a CPU int32 matmul (C_D from bridger_path_matrix, pinned by
  exhaustive enumeration in test_boundary_cpu.py), bitwise, on random 0/1 P;
* end to end, for both the fused K5 kernel (variant "gemm": decisions never
  leave shared memory, a4 folded into the contraction) and the staged
  K1 -> K2 -> K3 pipeline (variant "gemm_staged"): labels / scores / raw
  accumulators == oracle (same bar as the traversal).
"""
import numpy as np
import pytest

import oracle
from synth import gen_x, inject_specials, make_config, perfect_ensemble, prune_ensemble
from synth.trees import ModelDesc
from tests.test_gpu_parity import check, dev

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
import paper_2405_12491_b200 as B  # noqa: E402


def cpu_decisions(m, X, t):
    """a1+a2 by definition, from the ORIGINAL node arrays of a perfect,
    heap-ordered tree (independent of the library's lowering): decision i =
    [x[feature_i] <= threshold_i], NaN -> missing_left_i."""
    tr = m.tree(t)
    left, right = np.asarray(tr["left"]), np.asarray(tr["right"])
    # heap position of every internal node (children of heap h: 2h+1, 2h+2),
    # by a walk from the root over the original child links (any node order)
    heap, order = {0: 0}, [0]
    for n in order:
        if left[n] != -1:
            heap[int(left[n])], heap[int(right[n])] = 2 * heap[n] + 1, 2 * heap[n] + 2
            order += [int(left[n]), int(right[n])]
    inner = [n for n in order if left[n] != -1]
    I = len(inner)
    D = int(np.log2(I + 1))
    assert I == (1 << D) - 1 and sorted(heap[n] for n in inner) == list(range(I)), "perfect tree"
    ip, _ = B.gemm_geometry(max(D, 1))
    feat = np.zeros(I, np.int64)
    thr = np.zeros(I, np.float32)
    ml = np.zeros(I, np.uint8)
    for n in inner:
        feat[heap[n]] = tr["feature"][n]
        thr[heap[n]] = tr["threshold"][n]
        if tr["missing_left"] is not None:
            ml[heap[n]] = tr["missing_left"][n]
    x = X[:, feat]
    with np.errstate(invalid="ignore"):
        d = (x <= thr[None, :])
    d |= np.isnan(x) & (ml[None, :] != 0)
    out = np.zeros((X.shape[0], ip), np.int8)
    out[:, :I] = d
    return out


@pytest.mark.parametrize("name,ml", [("C2", False), ("C3", False), ("mixed", True)])
def test_k1_decisions_bitwise(name, ml):
    if name == "mixed":
        m = perfect_ensemble(21, 10, 6, 9, kind="classification", n_classes=3, calib_rows=512)
        m = prune_ensemble(m, 21, p=0.0, with_missing=ml)
        X = inject_specials(gen_x(22, 0, 1001, 9), 22, rate=0.05)
    else:
        c, m = make_config(name, n_trees=12)
        X = gen_x(c.seed, 0, 1001, c.n_features)
    g = B.Model(m)
    D = int(np.log2(int(np.sum(np.asarray(m.tree(0)["left"]) != -1)) + 1))
    ip, _ = B.gemm_geometry(D)
    P = g.step_decisions(dev(X), 2, 5, ip).cpu().numpy()
    for j in range(5):
        np.testing.assert_array_equal(P[j], cpu_decisions(m, X, 2 + j))


@pytest.mark.parametrize("D", [3, 6, 8])
def test_k2_path_contraction_is_int_matmul(D):
    m = perfect_ensemble(23, 4, D, 5, kind="regression")
    g = B.Model(m)
    ip, lp = B.gemm_geometry(D)
    rows = 1000  # 7 full 128-row tiles + a ragged tail
    rng = np.random.default_rng(D)
    P = (rng.random((rows, ip)) < 0.5).astype(np.int8)
    S = g.step_path_scores(D, dev(P)).cpu().numpy()
    Cm, _ = B.path_matrix(D)
    ref = P.astype(np.int32) @ Cm.astype(np.int32)
    np.testing.assert_array_equal(S, ref)


@pytest.mark.parametrize("D", [3, 6, 7, 8])
def test_k2_sparse_path_contraction_is_int_matmul(D):
    """K2s (tcgen05.mma.sp kind::i8, 2:4-sparse C_sp^T as operand A) equals a
    CPU int32 matmul with the regrouped path matrix, bitwise, on random 0/1
    decisions in the sparse K order (pad positions random too: C_sp is zero
    there), 7 full 128-row tiles + a ragged tail."""
    m = perfect_ensemble(23, 4, D, 5, kind="regression")
    g = B.Model(m)
    _, lp = B.gemm_geometry(D)
    Csp = B.path_matrix_sparse(D)
    rows = 1000
    rng = np.random.default_rng(100 + D)
    P = (rng.random((rows, Csp.shape[0])) < 0.5).astype(np.int8)
    S = g.step_path_scores_sparse(D, dev(P)).cpu().numpy()
    ref = P.astype(np.int32) @ Csp[:, :lp].astype(np.int32)
    np.testing.assert_array_equal(S, ref)


@pytest.mark.parametrize("variant", ["gemm", "gemm_staged", "gemm_sparse"])
@pytest.mark.parametrize("name,rows", [("C1", None), ("C2", 9001), ("C3", 5001)])
def test_gemm_variant_end_to_end(name, rows, variant):
    c, m = make_config(name, n_trees=None if name != "C3" else 120)
    if name == "C1":
        from synth import iris_like_x
        X = iris_like_x(1)
    else:
        X = gen_x(c.seed, 0, rows, c.n_features)
    g, _ = check(m, X, variant=variant, apply=False)
    assert g.info()["variant"] == variant


@pytest.mark.parametrize("variant", ["gemm", "gemm_staged", "gemm_sparse"])
def test_gemm_variant_pruned_missing_mixed_depth(variant):
    m = perfect_ensemble(25, 40, 7, 13, kind="classification", n_classes=4, calib_rows=1024)
    m = prune_ensemble(m, 25, p=0.2, with_missing=True)
    X = inject_specials(gen_x(26, 0, 3001, 13), 26, rate=0.02)
    check(m, X, variant=variant, apply=False)


@pytest.mark.parametrize("D", [1, 2, 3, 4, 5, 6, 7, 8])
def test_fused_every_depth(D):
    # every K5 geometry (I_pad 32..256, L_pad 16..256, popc row I), ragged last tile
    m = perfect_ensemble(40 + D, 9, D, 11, kind="classification", n_classes=3, calib_rows=512)
    X = inject_specials(gen_x(60 + D, 0, 777, 11), 60 + D, rate=0.01)
    check(m, X, variant="gemm", apply=False)


@pytest.mark.parametrize("D", [1, 2, 4, 5, 7, 8])
def test_sparse_variant_every_depth(D):
    # every K2s geometry (k_sp 64..256, one or two 128-leaf M-tiles), ragged last tile
    m = perfect_ensemble(80 + D, 7, D, 11, kind="classification", n_classes=3, calib_rows=512)
    X = inject_specials(gen_x(90 + D, 0, 1777, 11), 90 + D, rate=0.01)
    check(m, X, variant="gemm_sparse", apply=False)


def test_sparse_matches_dense_staged_bitwise():
    c, m = make_config("C2")
    X = dev(gen_x(2, 0, 30000, 28))
    a = B.Model(m, variant="gemm_sparse").predict_raw(X).cpu().numpy()
    b = B.Model(m, variant="gemm_staged").predict_raw(X).cpu().numpy()
    np.testing.assert_array_equal(a, b)


def test_fused_many_tiles_per_cta_regression():
    # > 148 tiles: each persistent CTA walks several row tiles (accumulators reset
    # per tile), GBDT SUM aggregation, E53 bitwise
    m = perfect_ensemble(71, 30, 6, 17, kind="regression", calib_rows=1024)
    check(m, gen_x(72, 0, 148 * 128 * 2 + 77, 17), variant="gemm", apply=False)


def test_fused_multiclass_k8_and_fp64_tier():
    m = perfect_ensemble(73, 25, 5, 12, kind="classification", n_classes=8, calib_rows=512)
    check(m, gen_x(74, 0, 4099, 12), variant="gemm", apply=False)
    # subnormal leaf values force the fp64 accumulation tier (reading c9): rtol 1e-5
    v = m.value.copy()
    v[::7] = np.float32(1e-40)
    m2 = ModelDesc(**{**m.__dict__, "value": v})
    g = B.Model(m2, variant="gemm")
    assert g.info()["exact_tier"] == "F64"
    check(m2, gen_x(74, 0, 2001, 12), variant="gemm", exact=False, apply=False)


def test_fused_matches_staged_bitwise_full_c2_block():
    # the two GEMM-form pipelines agree bit for bit on raw int64 accumulators
    c, m = make_config("C2")
    X = dev(gen_x(2, 0, 50000, 28))
    a = B.Model(m, variant="gemm").predict_raw(X).cpu().numpy()
    b = B.Model(m, variant="gemm_staged").predict_raw(X).cpu().numpy()
    np.testing.assert_array_equal(a, b)

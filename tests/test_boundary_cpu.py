"""C-ABI boundary and host lowering, no GPU needed.

* libbridger.so loads and exports every symbol include/bridger.h declares;
* step a0 lowering: the universal path matrix against its closed form and by
  exhaustive enumeration of all 2^I decision vectors for D <= 4 (exactly one
  leaf satisfies P.C_D == D_D and it is the leaf the decisions route to);
* padding by leaf replication preserves every walk (checked with the oracle on
  the padded heap tree vs the original tree, NaN rows included);
* validation rejects each class of malformed tree; exactness tiers.
"""
import itertools
import os
import re

import numpy as np
import pytest

import oracle
import paper_2405_12491_b200 as B
from synth import multiclass_gbdt, gen_x, inject_specials, make_config, perfect_ensemble, prune_ensemble
from synth.trees import ModelDesc

HDR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "bridger.h")


def test_library_exports_every_declared_symbol():
    src = open(HDR).read()
    declared = set(re.findall(r"^(?:bridger_status|const char\s*\*|int32_t|int64_t)\s+(bridger_\w+)\(", src, re.M))
    assert len(declared) >= 20
    lib = B.lib()
    for name in sorted(declared):
        assert hasattr(lib, name), name
    assert declared == set(B.EXPORTS)


@pytest.mark.parametrize("D", [1, 2, 3, 4, 5, 6, 7, 8])
def test_path_matrix_closed_form(D):
    Cm, Dv = B.path_matrix(D)
    I, L = (1 << D) - 1, 1 << D
    ip, lp = B.gemm_geometry(D)
    assert Cm.shape == (ip, lp) and ip % 32 == 0 and lp % 16 == 0 and ip >= I and lp >= L
    assert np.all(Cm[I:] == 0) and np.all(Cm[:, L:] == 0)
    for l in range(L):
        assert Dv[l] == D - bin(l).count("1")
        # column l has exactly D non-zeros: its ancestors, +1 where the path turns left
        assert np.count_nonzero(Cm[:I, l]) == D
    for i in range(I):
        # node i at depth d covers 2^(D-d) leaves: half +1 (left subtree), half -1
        d = int(np.floor(np.log2(i + 1)))
        assert np.sum(Cm[i] == 1) == np.sum(Cm[i] == -1) == 1 << (D - d - 1)


@pytest.mark.parametrize("D", [1, 2, 3, 4])
def test_path_matrix_exhaustive_enumeration(D):
    Cm, Dv = B.path_matrix(D)
    I, L = (1 << D) - 1, 1 << D
    Cc = Cm[:I, :L].astype(np.int32)
    for bits in itertools.product([0, 1], repeat=I):
        P = np.array(bits, np.int32)           # P[i] = 1 <=> decision "x <= t" (go left) at heap node i
        S = P @ Cc
        hits = np.nonzero(S == Dv)[0]
        i = 0
        for _ in range(D):
            i = 2 * i + 1 + (1 - P[i])
        assert hits.tolist() == [i - I]


def _padded_as_desc(m, K):
    """Turn each tree's padded heap form into plain node arrays (test-side)."""
    offs, F_, T_, L_, R_, V_, M_, ids = [0], [], [], [], [], [], [], []
    for t in range(m.n_trees):
        p = B.lower_tree(m, t)
        D = p["depth"]
        I, L = (1 << D) - 1, 1 << D
        n = I + L
        f = np.zeros(n, np.int32); th = np.zeros(n, np.float32); ml = np.zeros(n, np.uint8)
        lf = np.full(n, -1, np.int32); rt = np.full(n, -1, np.int32); v = np.zeros((n, K), np.float32)
        f[:I] = p["feature"]; th[:I] = p["threshold"]; ml[:I] = p["missing_left"]
        lf[:I] = 2 * np.arange(I) + 1; rt[:I] = 2 * np.arange(I) + 2
        v[I:] = p["leaf_value"]
        offs.append(offs[-1] + n); F_.append(f); T_.append(th); L_.append(lf); R_.append(rt)
        V_.append(v.reshape(-1)); M_.append(ml); ids.append(p["leaf_id"])
    d = ModelDesc(n_features=m.n_features, n_outputs=K, tree_offsets=np.asarray(offs, np.int64),
                  feature=np.concatenate(F_), threshold=np.concatenate(T_), left=np.concatenate(L_),
                  right=np.concatenate(R_), value=np.concatenate(V_),
                  missing_left=np.concatenate(M_) if m.missing_left is not None else None,
                  task=m.task, agg=m.agg, post=m.post, base_score=m.base_score, leaf_scale=m.leaf_scale)
    return d, ids


@pytest.mark.parametrize("ml", [False, True])
def test_padding_preserves_walk(ml):
    m = perfect_ensemble(3, 12, 5, 6, kind="classification", n_classes=3, calib_rows=512)
    m = prune_ensemble(m, 3, p=0.25, with_missing=ml)
    X = inject_specials(gen_x(4, 0, 600, 6), 4, rate=0.05)
    pd, ids = _padded_as_desc(m, 3)
    a = oracle.run(m, X)
    b = oracle.run(pd, X)
    np.testing.assert_array_equal(a["acc"], b["acc"])
    I_of = [(1 << B.lower_tree(m, t)["depth"]) - 1 for t in range(m.n_trees)]
    for t in range(m.n_trees):
        np.testing.assert_array_equal(a["leaf"][:, t], ids[t][b["leaf"][:, t] - I_of[t]])


def _bad(m, **kw):
    d = ModelDesc(**{**m.__dict__, **kw})
    with pytest.raises(B.BridgerError) as ei:
        B.validate(d)
    return ei.value.status


def test_validation_rejects_malformed_trees():
    _, m = make_config("C1")
    B.validate(m)
    l = m.left.copy(); l[0] = -1
    assert _bad(m, left=l) == B.E_INVALID_TREE               # one child -1
    l = m.left.copy(); l[1] = 1
    assert _bad(m, left=l) == B.E_INVALID_TREE               # self loop
    l = m.left.copy(); l[0] = 99
    assert _bad(m, left=l) == B.E_INVALID_TREE               # out of range
    r = m.right.copy(); r[1] = m.left[1]
    assert _bad(m, right=r) == B.E_INVALID_TREE              # l == r
    l = m.left.copy(); l[2] = m.left[1]; r = m.right.copy(); r[2] = m.right[1]
    assert _bad(m, left=l, right=r) == B.E_INVALID_TREE      # two parents / unreachable
    f = m.feature.copy(); f[0] = 4
    assert _bad(m, feature=f) == B.E_INVALID_TREE            # feature >= F
    t = m.threshold.copy(); t[0] = np.nan
    assert _bad(m, threshold=t) == B.E_INVALID_TREE          # NaN threshold
    v = m.value.copy(); v[-1] = np.inf
    assert _bad(m, value=v) == B.E_INVALID_TREE              # non-finite leaf
    o = m.tree_offsets.copy(); o[-1] = 0
    assert _bad(m, tree_offsets=o) == B.E_INVALID_TREE       # offsets not increasing
    assert _bad(m, n_outputs=0) == B.E_SHAPE
    assert _bad(m, post=1) == B.E_UNSUPPORTED                # sigmoid on K=3
    mr = make_config("C3", n_trees=4)[1]
    assert _bad(mr, post=2) == B.E_UNSUPPORTED               # softmax on a regressor
    mc = multiclass_gbdt(7, 2, 3, 5, 3)
    B.validate(mc)
    assert _bad(mc, n_outputs=1, post=0) == B.E_SHAPE        # tree_output >= K
    to = mc.tree_output.copy(); to[0] = -1
    assert _bad(mc, tree_output=to) == B.E_SHAPE
    vv = mc.value.copy(); vv[np.flatnonzero(mc.left == -1)[0]] = np.nan
    assert _bad(mc, value=vv) == B.E_INVALID_TREE            # scalar leaves checked at width 1


def test_multiclass_lowering_expands_scalar_leaves():
    # reading c15: a tree with tree_output k lowers to K-vector leaves that are
    # zero outside column k, carrying its scalar leaf values in column k
    mc = multiclass_gbdt(8, 3, 4, 6, 4)
    for t in range(mc.n_trees):
        p = B.lower_tree(mc, t)
        k = int(mc.tree_output[t])
        lv = p["leaf_value"]
        assert lv.shape == (16, 4)
        np.testing.assert_array_equal(np.delete(lv, k, axis=1), 0.0)
        a = int(mc.tree_offsets[t])
        np.testing.assert_array_equal(lv[:, k], mc.value[a + p["leaf_id"]])


def _lsb_exp(v):
    v = np.float64(v)
    m, e = np.frexp(abs(v))                 # v = m 2^e, m in [0.5,1)
    mi = int(m * 2 ** 53)
    tz = (mi & -mi).bit_length() - 1
    return e - 53 + tz


def test_exactness_tiers_match_definition():
    for name in ("C1", "C2", "C3"):
        _, m = make_config(name, n_trees=50 if name != "C1" else None)
        q, tier, l2 = B.analyze_exactness(m)
        K = m.n_outputs
        leaves = m.left == -1
        vals = m.value.reshape(-1, K)[leaves]
        nz = vals[vals != 0]
        assert q == min(_lsb_exp(v) for v in nz)
        tree_of = np.repeat(np.arange(m.n_trees), np.diff(m.tree_offsets))[leaves]
        Mk = [sum(int(np.max(np.abs(vals[tree_of == t, k]).astype(np.float64)) * 2.0 ** -q)
                  for t in range(m.n_trees)) for k in range(K)]
        assert abs(np.log2(max(Mk)) - l2) < 1e-9
        assert tier == ("E53" if max(Mk) < 2 ** 53 else "E63" if max(Mk) < 2 ** 63 else "F64")
    m = make_config("C1")[1]
    v = m.value.copy(); v[-1] = 1.4e-45                      # subnormal -> q = -149 -> M >= 2^63
    assert B.analyze_exactness(ModelDesc(**{**m.__dict__, "value": v}))[1] == "F64"


def test_no_fallback_without_library(tmp_path):
    """The product path fails loudly without its CUDA library: a copy of the
    package with no libbridger.so refuses to import (no CPU fallback)."""
    import shutil
    import subprocess
    import sys
    pkg = os.path.dirname(B.__file__)
    dst = tmp_path / "paper_2405_12491_b200"
    shutil.copytree(pkg, dst, ignore=shutil.ignore_patterns("*.so", "build", "__pycache__", "csrc"))
    r = subprocess.run([sys.executable, "-c", "import paper_2405_12491_b200"], cwd=tmp_path,
                       capture_output=True, text=True)
    assert r.returncode != 0
    assert "libbridger" in (r.stderr + r.stdout)


@pytest.mark.skipif(__import__("torch").cuda.is_available(), reason="checks the no-device error path")
def test_no_device_is_a_cuda_error():
    """Without a GPU, loading a model returns BRIDGER_E_CUDA (the oracle is
    never consulted)."""
    c, m = make_config("C1")
    with pytest.raises(B.BridgerError) as ei:
        B.Model(m, device=0)
    assert ei.value.status == B.E_CUDA


def test_variant_table_header_matches_measurement():
    """AUTO's per-depth table (csrc/variant_table.h) is the one generated from
    the committed measurement profiles/variant_table.json (best variant per
    depth of a 1M-row x 100-tree forest on B200)."""
    import json
    import os
    import re
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    d = json.load(open(os.path.join(root, "profiles", "variant_table.json")))
    hdr = open(os.path.join(root, "paper_2405_12491_b200", "csrc", "variant_table.h")).read()
    vals = [int(v) for v in re.search(r"kVariantByDepth\[16\] = \{([^}]*)\}", hdr).group(1).split(",")]
    code = {"traverse": 1, "gemm": 2, "gemm_staged": 3, "gemm_sparse": 4}
    for r in d["rows"]:
        assert vals[r["depth"]] == code[r["best"]]
        ms = {k: r[k + "_ms"] for k in code if k + "_ms" in r}
        assert r["best"] == min(ms, key=ms.get)


def test_sparse_path_matrix_regrouping_is_2_4_structured():
    """bridger_path_matrix_sparse: the dense C_D (pinned by exhaustive
    enumeration above) with heap node i moved to K position i + [i >= 3]; every
    group of 4 consecutive K positions holds <= 2 non-zeros of any leaf column
    (2:4 structured sparsity, the operand form of tcgen05.mma.sp), zero rows
    at the pads, and every leaf keeps exactly its D ancestors."""
    for D in range(1, 9):
        Cs = B.path_matrix_sparse(D)
        Cd, _ = B.path_matrix(D)
        I, L = (1 << D) - 1, 1 << D
        assert Cs.shape == ((((1 << D) + 63) // 64) * 64, (((1 << D) + 127) // 128) * 128)
        pos = [i + (1 if i >= 3 else 0) for i in range(I)]
        np.testing.assert_array_equal(Cs[pos, :L], Cd[:I, :L])
        mask = np.ones(Cs.shape[0], bool)
        mask[pos] = False
        assert not Cs[mask].any() and not Cs[:, L:].any()
        nz = (Cs != 0).reshape(Cs.shape[0] // 4, 4, Cs.shape[1]).sum(axis=1)
        assert nz.max() <= 2
        assert ((Cs != 0).sum(axis=0)[:L] == D).all()

"""CPU oracle -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import this package.  The product path
(``paper_2405_12491_b200``) never imports it and shares no code with it.

``oracle.c`` is a plain node-by-node walker over the original node arrays in
fp64; see its header for the definition and the paper
passages it follows.  Pins (tests/test_oracle_*.py): SPEC.md:286/288 worked
examples and a hand-computed iris-shaped tree (tests/golden/), a brute-force
region oracle on tiny trees, scikit-learn's own ``apply``/``predict`` (a library
routine), and invariants.  The sigmoid probability of binary GBDT is "parity
unpinned" beyond the 1e-5 tolerance (reading c10).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle.c")


def build(force: bool = False) -> str:
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math",
                               "-fPIC", "-shared", "-pthread", _SRC, "-o", _SO, "-lm"])
    return _SO


class _Model(C.Structure):
    _fields_ = [("n_trees", C.c_int32), ("n_features", C.c_int32), ("n_outputs", C.c_int32),
                ("tree_offsets", C.c_void_p), ("feature", C.c_void_p), ("threshold", C.c_void_p),
                ("left", C.c_void_p), ("right", C.c_void_p), ("value", C.c_void_p),
                ("missing_left", C.c_void_p), ("task", C.c_int32), ("agg", C.c_int32),
                ("post", C.c_int32), ("base_score", C.c_void_p), ("leaf_scale", C.c_double),
                ("tree_output", C.c_void_p)]


_lib = None


def _load():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _lib.oracle_run.restype = C.c_int
        _lib.oracle_run.argtypes = [C.POINTER(_Model), C.c_void_p, C.c_int64, C.c_int32, C.c_int,
                                    C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                    C.c_void_p]
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data


def n_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def run(m, X: np.ndarray, n_threads: int | None = None, want=("leaf", "acc", "s", "label", "proba", "pred")):
    """Walk every row of X through model ``m`` (a synth.ModelDesc or any object
    with the same array attributes).  Returns a dict with the requested outputs:
    leaf [n,T] int32 (original tree-local ids), acc [n,K] fp64 raw sums, s [n,K]
    fp64 final scores, label [n] int32, proba [n,C] fp32, pred [n,K] fp32."""
    lib = _load()
    X = np.ascontiguousarray(X, dtype=np.float32)
    n, F = X.shape
    T, K = len(m.tree_offsets) - 1, int(m.n_outputs)
    keep = dict(offs=np.ascontiguousarray(m.tree_offsets, np.int64),
                feat=np.ascontiguousarray(m.feature, np.int32),
                thr=np.ascontiguousarray(m.threshold, np.float32),
                l=np.ascontiguousarray(m.left, np.int32), r=np.ascontiguousarray(m.right, np.int32),
                v=np.ascontiguousarray(m.value, np.float32),
                ml=None if m.missing_left is None else np.ascontiguousarray(m.missing_left, np.uint8),
                base=None if m.base_score is None else np.ascontiguousarray(m.base_score, np.float64),
                tout=None if getattr(m, "tree_output", None) is None else np.ascontiguousarray(m.tree_output, np.int32))
    mm = _Model(T, int(m.n_features), K, _ptr(keep["offs"]), _ptr(keep["feat"]), _ptr(keep["thr"]),
                _ptr(keep["l"]), _ptr(keep["r"]), _ptr(keep["v"]), _ptr(keep["ml"]), int(m.task),
                int(m.agg), int(m.post), _ptr(keep["base"]), float(m.leaf_scale), _ptr(keep["tout"]))
    classif = int(m.task) == 1
    Cp = (2 if K == 1 else K)
    out = dict(
        leaf=np.empty((n, T), np.int32) if "leaf" in want else None,
        acc=np.empty((n, K), np.float64) if "acc" in want else None,
        s=np.empty((n, K), np.float64) if "s" in want else None,
        label=np.empty(n, np.int32) if (classif and "label" in want) else None,
        proba=np.empty((n, Cp), np.float32) if (classif and "proba" in want) else None,
        pred=np.empty((n, K), np.float32) if (not classif and "pred" in want) else None)
    rc = lib.oracle_run(C.byref(mm), X.ctypes.data, n, F, n_threads or n_cores(),
                        _ptr(out["leaf"]), _ptr(out["acc"]), _ptr(out["s"]), _ptr(out["label"]),
                        _ptr(out["proba"]), _ptr(out["pred"]))
    if rc != 0:
        raise ValueError(f"oracle_run failed with code {rc}")
    return {k: v for k, v in out.items() if v is not None}


class _Linear(C.Structure):
    _fields_ = [("n_features", C.c_int32), ("n_outputs", C.c_int32), ("coef", C.c_void_p),
                ("intercept", C.c_void_p), ("mean", C.c_void_p), ("scale", C.c_void_p),
                ("task", C.c_int32), ("post", C.c_int32)]


def run_linear(m, X: np.ndarray):
    """Linear model (oracle.c oracle_linear_run): ``m`` has n_features, n_outputs,
    coef [K,F] fp64, intercept [K] | None, mean/scale [F] | None (StandardScaler),
    task, post.  Returns s [n,K] fp64 and label/proba (classification) or pred."""
    lib = _load()
    if not hasattr(lib, "_lin_ready"):
        lib.oracle_linear_run.restype = C.c_int
        lib.oracle_linear_run.argtypes = [C.POINTER(_Linear), C.c_void_p, C.c_int64, C.c_int32,
                                          C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        lib._lin_ready = True
    X = np.ascontiguousarray(X, dtype=np.float32)
    n, F = X.shape
    K = int(m.n_outputs)
    keep = dict(coef=np.ascontiguousarray(m.coef, np.float64).reshape(K, F),
                b=None if m.intercept is None else np.ascontiguousarray(m.intercept, np.float64),
                mean=None if m.mean is None else np.ascontiguousarray(m.mean, np.float64),
                scale=None if m.scale is None else np.ascontiguousarray(m.scale, np.float64))
    mm = _Linear(int(m.n_features), K, _ptr(keep["coef"]), _ptr(keep["b"]), _ptr(keep["mean"]),
                 _ptr(keep["scale"]), int(m.task), int(m.post))
    classif = int(m.task) == 1
    out = dict(s=np.empty((n, K), np.float64),
               label=np.empty(n, np.int32) if classif else None,
               proba=np.empty((n, 2 if K == 1 else K), np.float32) if classif else None,
               pred=None if classif else np.empty((n, K), np.float32))
    rc = lib.oracle_linear_run(C.byref(mm), X.ctypes.data, n, F, _ptr(out["s"]), _ptr(out["label"]),
                               _ptr(out["proba"]), _ptr(out["pred"]))
    if rc != 0:
        raise ValueError(f"oracle_linear_run failed with code {rc}")
    return {k: v for k, v in out.items() if v is not None}

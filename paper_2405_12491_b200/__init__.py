"""paper_2405_12491_b200 -- B200-native tree-ensemble inference (the CML hot
path of arxiv 2405.12491, "bridger").

Thin Python binding over ``libbridger.so`` (C ABI in ``include/bridger.h``).
This module only marshals arguments: every compute step runs in the library's
sm_100a CUDA kernels.  PyTorch is used for device memory and streams only.
There is no CPU fallback: if the shared library is missing, importing this
package raises (build it with ``__graft_entry__.build()`` or
``python paper_2405_12491_b200/build.py``).
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libbridger.so")

OK, E_NULL_ARG, E_SHAPE, E_INVALID_TREE, E_UNSUPPORTED, E_CUDA, E_OOM = range(7)
VARIANTS = {"auto": 0, "traverse": 1, "gemm": 2, "gemm_staged": 3, "gemm_sparse": 4}
TIERS = {0: "E53", 1: "E63", 2: "F64"}


class BridgerError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status


_STATUS = {0: "BRIDGER_OK", 1: "BRIDGER_E_NULL_ARG", 2: "BRIDGER_E_SHAPE", 3: "BRIDGER_E_INVALID_TREE",
           4: "BRIDGER_E_UNSUPPORTED", 5: "BRIDGER_E_CUDA", 6: "BRIDGER_E_OOM"}


class _Desc(C.Structure):
    _fields_ = [("n_trees", C.c_int32), ("n_features", C.c_int32), ("n_outputs", C.c_int32),
                ("tree_offsets", C.c_void_p), ("feature", C.c_void_p), ("threshold", C.c_void_p),
                ("left", C.c_void_p), ("right", C.c_void_p), ("value", C.c_void_p),
                ("missing_left", C.c_void_p), ("task", C.c_int32), ("agg", C.c_int32), ("post", C.c_int32),
                ("base_score", C.c_void_p), ("leaf_scale", C.c_double),
                ("force_fixed_point", C.c_int32), ("forced_scale_exp", C.c_int32), ("forced_tier", C.c_int32),
                ("tree_output", C.c_void_p)]


EXPORTS = [
    "bridger_model_load", "bridger_model_free", "bridger_model_info", "bridger_model_set_variant",
    "bridger_model_variant", "bridger_predict", "bridger_predict_proba", "bridger_apply",
    "bridger_predict_raw", "bridger_finalize", "bridger_predict_host", "bridger_step_decisions",
    "bridger_step_path_scores", "bridger_gemm_geometry", "bridger_path_matrix", "bridger_lower_tree",
    "bridger_analyze_exactness", "bridger_validate", "bridger_last_error", "bridger_status_string",
    "bridger_launch_count", "bridger_hot_kernel_timing", "bridger_hot_kernel_time", "bridger_model_layout",
    "bridger_hot_kernel_time_by", "bridger_linear_load", "bridger_linear_free", "bridger_linear_predict",
    "bridger_linear_predict_proba", "bridger_linear_decision", "bridger_probe_smem_bandwidth",
    "bridger_path_matrix_sparse", "bridger_step_path_scores_sparse", "bridger_predict_raw_scatter",
    "bridger_bin_codes_host",
]


def _load_lib():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built; run __graft_entry__.build() (no CPU fallback exists)")
    lib = C.CDLL(LIB_PATH)
    vp, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
    sig = {
        "bridger_model_load": ([vp, C.c_int, vp], i32),
        "bridger_model_free": ([vp], i32),
        "bridger_model_info": ([vp, vp, vp, vp, vp], i32),
        "bridger_model_set_variant": ([vp, i32], i32),
        "bridger_model_variant": ([vp], i32),
        "bridger_predict": ([vp, vp, i64, i32, vp, vp], i32),
        "bridger_predict_proba": ([vp, vp, i64, i32, vp, vp], i32),
        "bridger_apply": ([vp, vp, i64, i32, vp, vp], i32),
        "bridger_predict_raw": ([vp, vp, i64, i32, vp, vp], i32),
        "bridger_finalize": ([vp, vp, i64, i32, vp, i32, vp], i32),
        "bridger_predict_host": ([vp, vp, i64, i32, vp, i32], i32),
        "bridger_step_decisions": ([vp, vp, i64, i32, i32, i32, vp, vp], i32),
        "bridger_step_path_scores": ([vp, i32, vp, i64, vp, vp], i32),
        "bridger_gemm_geometry": ([i32, vp, vp], i32),
        "bridger_path_matrix": ([i32, vp, vp], i32),
        "bridger_lower_tree": ([vp, i32, vp, vp, vp, vp, vp, vp], i32),
        "bridger_analyze_exactness": ([vp, vp, vp, vp], i32),
        "bridger_validate": ([vp], i32),
        "bridger_last_error": ([], C.c_char_p),
        "bridger_status_string": ([i32], C.c_char_p),
        "bridger_launch_count": ([], i64),
        "bridger_hot_kernel_timing": ([i32], i32),
        "bridger_hot_kernel_time": ([vp, vp], i32),
        "bridger_model_layout": ([vp, vp, vp, vp, vp, vp], i32),
        "bridger_hot_kernel_time_by": ([i32, vp, vp], i32),
        "bridger_linear_load": ([vp, i32, vp], i32),
        "bridger_linear_free": ([vp], i32),
        "bridger_linear_predict": ([vp, vp, i64, i32, vp, vp], i32),
        "bridger_linear_predict_proba": ([vp, vp, i64, i32, vp, vp], i32),
        "bridger_linear_decision": ([vp, vp, i64, i32, vp, vp], i32),
        "bridger_probe_smem_bandwidth": ([i32, vp, vp], i32),
        "bridger_path_matrix_sparse": ([i32, vp, vp, vp], i32),
        "bridger_step_path_scores_sparse": ([vp, i32, vp, i64, vp, vp], i32),
        "bridger_predict_raw_scatter": ([vp, vp, i64, i32, vp, i32, i64, vp], i32),
        "bridger_bin_codes_host": ([vp, vp, i64, i32, i32, vp, vp], i32),
    }
    for name, (args, res) in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    return lib


_lib = _load_lib()


def lib():
    return _lib


def _check(status: int):
    if status != OK:
        raise BridgerError(status, _lib.bridger_last_error().decode(errors="replace"))


def launch_count() -> int:
    """Kernel launches issued by this thread through the library."""
    return int(_lib.bridger_launch_count())


def hot_kernel_timing(enable: bool) -> None:
    _check(_lib.bridger_hot_kernel_timing(1 if enable else 0))


def hot_kernel_time(kernel: int = 0):
    """(summed ms, launches) since the last query of kernel id `kernel`:
    0 dominant (traversal / K2), 1 K1 gather-compare, 2 K3 leaf gather, 3 fused K5."""
    ms, n = C.c_double(), C.c_int64()
    _check(_lib.bridger_hot_kernel_time_by(int(kernel), C.byref(ms), C.byref(n)))
    return ms.value, n.value


def probe_smem_bandwidth(device: int = 0):
    """(conflict-free, random) shared-memory LDS.64 GB/s measured now on `device`."""
    a, b = C.c_double(), C.c_double()
    _check(_lib.bridger_probe_smem_bandwidth(int(device), C.byref(a), C.byref(b)))
    return a.value, b.value


class _DescKeep:
    """A bridger_model_desc plus the numpy arrays it points into."""

    def __init__(self, m, force=None):
        self.arrs = dict(
            offs=np.ascontiguousarray(m.tree_offsets, np.int64),
            feat=np.ascontiguousarray(m.feature, np.int32),
            thr=np.ascontiguousarray(m.threshold, np.float32),
            l=np.ascontiguousarray(m.left, np.int32),
            r=np.ascontiguousarray(m.right, np.int32),
            v=np.ascontiguousarray(m.value, np.float32),
            ml=None if getattr(m, "missing_left", None) is None else np.ascontiguousarray(m.missing_left, np.uint8),
            base=None if getattr(m, "base_score", None) is None else np.ascontiguousarray(m.base_score, np.float64),
            tout=None if getattr(m, "tree_output", None) is None else np.ascontiguousarray(m.tree_output, np.int32),
        )
        a = self.arrs
        p = lambda x: None if x is None else x.ctypes.data
        self.desc = _Desc(len(a["offs"]) - 1, int(m.n_features), int(m.n_outputs), p(a["offs"]), p(a["feat"]),
                          p(a["thr"]), p(a["l"]), p(a["r"]), p(a["v"]), p(a["ml"]), int(getattr(m, "task", 0)),
                          int(getattr(m, "agg", 0)), int(getattr(m, "post", 0)), p(a["base"]),
                          float(getattr(m, "leaf_scale", 1.0)), 0, 0, 0, p(a["tout"]))
        if force is not None:
            self.desc.force_fixed_point = 1
            self.desc.forced_scale_exp = int(force[0])
            self.desc.forced_tier = int(force[1])

    @property
    def ptr(self):
        return C.byref(self.desc)


def _stream_ptr(device):
    """The caller's current CUDA stream on `device` (raw handle).  torch's
    private raw-stream getter costs ~0.2 us against ~2.3 us for
    torch.cuda.current_stream() -- a quarter of a small predict's host time."""
    import torch
    idx = device.index if device.index is not None else torch.cuda.current_device()
    raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)
    if raw is not None:
        return C.c_void_p(raw(idx))
    return C.c_void_p(torch.cuda.current_stream(device).cuda_stream)


# ----------------------------------------------------------- host helpers ---
def validate(m) -> None:
    k = _DescKeep(m)
    _check(_lib.bridger_validate(k.ptr))


def analyze_exactness(m):
    """(q, tier name, log2 M) of a model description (reading c9)."""
    k = _DescKeep(m)
    q, t, l2 = C.c_int32(), C.c_int32(), C.c_double()
    _check(_lib.bridger_analyze_exactness(k.ptr, C.byref(q), C.byref(t), C.byref(l2)))
    return q.value, TIERS[t.value], l2.value


def bin_codes_host(m, X, method: str):
    """Host emulation of the threshold-bin codes from the bucketed ("bucket")
    or bucket-entry ("entry") tables the load builds (bridger_bin_codes_host):
    (codes uint16 [n][F], NB), NB = 0 and codes None when that table is not
    built.  For CPU tests of the table construction."""
    import numpy as np
    k = _DescKeep(m)
    X = np.ascontiguousarray(X, dtype=np.float32)
    codes = np.zeros(X.shape, dtype=np.uint16)
    nb = C.c_int32()
    _check(_lib.bridger_bin_codes_host(k.ptr, X.ctypes.data, X.shape[0], X.shape[1], {"bucket": 1, "entry": 2}[method],
                                       codes.ctypes.data, C.byref(nb)))
    return (codes if nb.value else None), nb.value


def gemm_geometry(depth: int):
    ip, lp = C.c_int32(), C.c_int32()
    _check(_lib.bridger_gemm_geometry(depth, C.byref(ip), C.byref(lp)))
    return ip.value, lp.value


def path_matrix(depth: int):
    """(C [I_pad, L_pad] int8, Dv [2^D] int32) of the library's lowering."""
    ip, lp = gemm_geometry(depth)
    Cm = np.zeros((ip, lp), np.int8)
    Dv = np.zeros(1 << depth, np.int32)
    _check(_lib.bridger_path_matrix(depth, Cm.ctypes.data, Dv.ctypes.data))
    return Cm, Dv


def path_matrix_sparse(depth: int):
    """(C_sp [k_sp, m_sp] int8) -- the path matrix with K regrouped for 2:4
    sparsity (node i at K position i + [i >= 3]), as the library lowers it."""
    ks, ms = C.c_int32(), C.c_int32()
    _check(_lib.bridger_path_matrix_sparse(depth, None, C.byref(ks), C.byref(ms)))
    Cm = np.zeros((ks.value, ms.value), np.int8)
    _check(_lib.bridger_path_matrix_sparse(depth, Cm.ctypes.data, None, None))
    return Cm


def lower_tree(m, tree: int):
    """Padded perfect heap form of one tree, as the library lowers it."""
    k = _DescKeep(m)
    d = C.c_int32()
    _check(_lib.bridger_lower_tree(k.ptr, tree, C.byref(d), None, None, None, None, None))
    D = d.value
    I, L, K = (1 << D) - 1, 1 << D, int(m.n_outputs)
    feat = np.zeros(max(I, 1), np.int32)
    thr = np.zeros(max(I, 1), np.float32)
    ml = np.zeros(max(I, 1), np.uint8)
    lid = np.zeros(L, np.int32)
    val = np.zeros(L * K, np.float32)
    _check(_lib.bridger_lower_tree(k.ptr, tree, C.byref(d), feat.ctypes.data, thr.ctypes.data, ml.ctypes.data,
                                   lid.ctypes.data, val.ctypes.data))
    return dict(depth=D, feature=feat[:I], threshold=thr[:I], missing_left=ml[:I], leaf_id=lid,
                leaf_value=val.reshape(L, K))


# ------------------------------------------------------------------ model ---
class Model:
    """A tree ensemble lowered and resident on one CUDA device."""

    def __init__(self, desc, device: int = 0, variant: Optional[str] = None, force_fixed_point=None):
        import torch  # noqa: F401  (device memory / streams)
        self._keep = _DescKeep(desc, force_fixed_point)
        self._h = C.c_void_p()
        self.device = int(device)
        _check(_lib.bridger_model_load(self._keep.ptr, self.device, C.byref(self._h)))
        self.n_trees = self._keep.desc.n_trees
        self.n_features = int(desc.n_features)
        self.n_outputs = int(desc.n_outputs)
        self.task = int(getattr(desc, "task", 0))
        self.post = int(getattr(desc, "post", 0))
        if variant is not None:
            self.set_variant(variant)

    @classmethod
    def from_arrays(cls, *, n_features, n_outputs, tree_offsets, feature, threshold, left, right, value,
                    missing_left=None, task=0, agg=0, post=0, base_score=None, leaf_scale=1.0, tree_output=None,
                    device=0):
        from types import SimpleNamespace
        d = SimpleNamespace(n_features=n_features, n_outputs=n_outputs, tree_offsets=tree_offsets, feature=feature,
                            threshold=threshold, left=left, right=right, value=value, missing_left=missing_left,
                            task=task, agg=agg, post=post, base_score=base_score, leaf_scale=leaf_scale,
                            tree_output=tree_output)
        return cls(d, device=device)

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            _lib.bridger_model_free(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- info / config
    def info(self) -> dict:
        d, t, a, q = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
        _check(_lib.bridger_model_info(self._h, C.byref(d), C.byref(t), C.byref(a), C.byref(q)))
        return dict(max_depth=d.value, exact_tier=TIERS[t.value], acc_is_int64=bool(a.value), acc_scale_exp=q.value,
                    variant={v: k for k, v in VARIANTS.items()}[_lib.bridger_model_variant(self._h)])

    def layout(self) -> dict:
        n, c, g, w, gr = (C.c_int32() for _ in range(5))
        _check(_lib.bridger_model_layout(self._h, C.byref(n), C.byref(c), C.byref(g), C.byref(w), C.byref(gr)))
        return dict(n_chunks=n.value, coded=c.value in (1, 7, 8), sparse=c.value == 2,
                    format={0: "heap", 1: "codes", 2: "sparse", 3: "heap_pretransposed", 4: "hybrid", 6: "stream",
                            7: "stream_codes", 8: "codes_deep"}[c.value],
                    global_trees=bool(g.value),
                    n_warps=w.value, group=gr.value)

    def set_variant(self, name: str):
        _check(_lib.bridger_model_set_variant(self._h, VARIANTS[name]))

    # -- helpers
    def _x(self, X):
        import torch
        if not (isinstance(X, torch.Tensor) and X.is_cuda and X.dtype == torch.float32):
            raise TypeError("X must be a CUDA float32 tensor")
        if X.dim() != 2 or X.shape[1] != self.n_features:
            raise ValueError(f"X must be [n_rows, {self.n_features}]")
        if not X.is_contiguous():
            raise ValueError("X must be contiguous (row-major)")
        return X

    def _n_proba(self):
        return 2 if self.n_outputs == 1 else self.n_outputs

    def _acc_dtype(self):
        import torch
        return torch.int64 if self.info()["acc_is_int64"] else torch.float64

    # -- hot path
    def predict(self, X, out=None):
        import torch
        X = self._x(X)
        n = X.shape[0]
        if out is None:
            if self.task == 1:
                out = torch.empty(n, dtype=torch.int32, device=X.device)
            else:
                out = torch.empty((n, self.n_outputs), dtype=torch.float32, device=X.device)
        _check(_lib.bridger_predict(self._h, X.data_ptr(), n, X.shape[1], out.data_ptr(), _stream_ptr(X.device)))
        return out

    def predict_proba(self, X, out=None):
        import torch
        X = self._x(X)
        n = X.shape[0]
        if out is None:
            out = torch.empty((n, self._n_proba()), dtype=torch.float32, device=X.device)
        _check(_lib.bridger_predict_proba(self._h, X.data_ptr(), n, X.shape[1], out.data_ptr(),
                                          _stream_ptr(X.device)))
        return out

    def apply(self, X, out=None):
        import torch
        X = self._x(X)
        n = X.shape[0]
        if out is None:
            out = torch.empty((n, self.n_trees), dtype=torch.int32, device=X.device)
        _check(_lib.bridger_apply(self._h, X.data_ptr(), n, X.shape[1], out.data_ptr(), _stream_ptr(X.device)))
        return out

    def predict_raw(self, X, out=None):
        import torch
        X = self._x(X)
        n = X.shape[0]
        if out is None:
            out = torch.empty((n, self.n_outputs), dtype=self._acc_dtype(), device=X.device)
        _check(_lib.bridger_predict_raw(self._h, X.data_ptr(), n, X.shape[1], out.data_ptr(),
                                        _stream_ptr(X.device)))
        return out

    def predict_raw_scatter(self, X, dest_ptrs, rows_per_rank: int):
        """Fused tree-sharding reduce (bridger_predict_raw_scatter): add every
        row's int64 partial into dest_ptrs[row // rows_per_rank] (device
        pointers of the ranks' zeroed accumulator slices, own or peer)."""
        X = self._x(X)
        arr = (C.c_void_p * len(dest_ptrs))(*[C.c_void_p(int(d)) for d in dest_ptrs])
        _check(_lib.bridger_predict_raw_scatter(self._h, X.data_ptr(), X.shape[0], X.shape[1], arr, len(dest_ptrs),
                                                int(rows_per_rank), _stream_ptr(X.device)))

    def finalize(self, acc, total_trees: int, proba: bool = False, out=None):
        import torch
        n = acc.shape[0]
        if out is None:
            if proba:
                out = torch.empty((n, self._n_proba()), dtype=torch.float32, device=acc.device)
            elif self.task == 1:
                out = torch.empty(n, dtype=torch.int32, device=acc.device)
            else:
                out = torch.empty((n, self.n_outputs), dtype=torch.float32, device=acc.device)
        _check(_lib.bridger_finalize(self._h, acc.data_ptr(), n, int(total_trees), out.data_ptr(), int(proba),
                                     _stream_ptr(acc.device)))
        return out

    def predict_host(self, X, proba: bool = False, out=None):
        """End-to-end call on HOST buffers (numpy array or pinned CPU tensor)."""
        import torch
        if isinstance(X, np.ndarray):
            X = torch.from_numpy(np.ascontiguousarray(X, np.float32))
        n = X.shape[0]
        if out is None:
            if proba:
                out = torch.empty((n, self._n_proba()), dtype=torch.float32)
            elif self.task == 1:
                out = torch.empty(n, dtype=torch.int32)
            else:
                out = torch.empty((n, self.n_outputs), dtype=torch.float32)
        _check(_lib.bridger_predict_host(self._h, X.data_ptr(), n, X.shape[1], out.data_ptr(), int(proba)))
        return out

    # -- step-level entry points (parity of individual §8(a) rows)
    def step_decisions(self, X, tree0: int, n_trees: int, i_pad: int):
        import torch
        X = self._x(X)
        out = torch.empty((n_trees, X.shape[0], i_pad), dtype=torch.int8, device=X.device)
        _check(_lib.bridger_step_decisions(self._h, X.data_ptr(), X.shape[0], X.shape[1], tree0, n_trees,
                                           out.data_ptr(), _stream_ptr(X.device)))
        return out

    def step_path_scores_sparse(self, depth: int, P):
        """a3 on the 2:4-sparse tensor path (K2s): P [rows, k_sp] int8 in the
        sparse K order -> S [rows, l_pad] int32."""
        import torch
        _, lp = gemm_geometry(depth)
        rows = P.shape[0]
        out = torch.empty((rows, lp), dtype=torch.int32, device=P.device)
        _check(_lib.bridger_step_path_scores_sparse(self._h, depth, P.data_ptr(), rows, out.data_ptr(),
                                                    _stream_ptr(P.device)))
        return out

    def step_path_scores(self, depth: int, P):
        import torch
        ip, lp = gemm_geometry(depth)
        rows = P.numel() // ip
        out = torch.empty((rows, lp), dtype=torch.int32, device=P.device)
        _check(_lib.bridger_step_path_scores(self._h, depth, P.data_ptr(), rows, out.data_ptr(),
                                             _stream_ptr(P.device)))
        return out


__all__ = ["Model", "BridgerError", "validate", "analyze_exactness", "bin_codes_host", "path_matrix", "path_matrix_sparse", "lower_tree",
           "gemm_geometry", "launch_count", "lib", "LIB_PATH", "EXPORTS"]


# ------------------------------------------------------------ linear models --
class _LinDesc(C.Structure):
    _fields_ = [("n_features", C.c_int32), ("n_outputs", C.c_int32), ("coef", C.c_void_p),
                ("intercept", C.c_void_p), ("scaler_mean", C.c_void_p), ("scaler_scale", C.c_void_p),
                ("task", C.c_int32), ("post", C.c_int32)]


class LinearModel:
    """A linear model on the device (bridger_linear_*): argument
    marshalling only.  ``m`` has n_features, n_outputs, coef [K,F], intercept [K] | None,
    mean / scale [F] | None (StandardScaler), task, post."""

    def __init__(self, m, device: int = 0):
        self.n_features, self.n_outputs = int(m.n_features), int(m.n_outputs)
        self.task, self.post = int(m.task), int(m.post)
        K, F = self.n_outputs, self.n_features
        keep = dict(coef=np.ascontiguousarray(m.coef, np.float64).reshape(K, F),
                    b=None if getattr(m, "intercept", None) is None else np.ascontiguousarray(m.intercept, np.float64),
                    mean=None if getattr(m, "mean", None) is None else np.ascontiguousarray(m.mean, np.float64),
                    scale=None if getattr(m, "scale", None) is None else np.ascontiguousarray(m.scale, np.float64))
        p = lambda x: None if x is None else x.ctypes.data
        d = _LinDesc(F, K, p(keep["coef"]), p(keep["b"]), p(keep["mean"]), p(keep["scale"]), self.task, self.post)
        self._h = C.c_void_p()
        _check(_lib.bridger_linear_load(C.byref(d), int(device), C.byref(self._h)))

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            _lib.bridger_linear_free(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _x(self, X):
        import torch
        if not (isinstance(X, torch.Tensor) and X.is_cuda and X.dtype == torch.float32 and X.is_contiguous()):
            raise TypeError("X must be a contiguous CUDA float32 tensor")
        if X.dim() != 2 or X.shape[1] != self.n_features:
            raise ValueError(f"X must be [n_rows, {self.n_features}]")
        return X

    def predict(self, X, out=None):
        import torch
        X = self._x(X)
        n = X.shape[0]
        if out is None:
            out = (torch.empty(n, dtype=torch.int32, device=X.device) if self.task == 1
                   else torch.empty((n, self.n_outputs), dtype=torch.float32, device=X.device))
        _check(_lib.bridger_linear_predict(self._h, X.data_ptr(), n, X.shape[1], out.data_ptr(), _stream_ptr(X.device)))
        return out

    def predict_proba(self, X, out=None):
        import torch
        X = self._x(X)
        n = X.shape[0]
        if out is None:
            out = torch.empty((n, 2 if self.n_outputs == 1 else self.n_outputs), dtype=torch.float32, device=X.device)
        _check(_lib.bridger_linear_predict_proba(self._h, X.data_ptr(), n, X.shape[1], out.data_ptr(),
                                                 _stream_ptr(X.device)))
        return out

    def decision_function(self, X, out=None):
        import torch
        X = self._x(X)
        n = X.shape[0]
        if out is None:
            out = torch.empty((n, self.n_outputs), dtype=torch.float64, device=X.device)
        _check(_lib.bridger_linear_decision(self._h, X.data_ptr(), n, X.shape[1], out.data_ptr(), _stream_ptr(X.device)))
        return out

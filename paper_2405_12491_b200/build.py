"""Build libbridger.so in-tree with nvcc for sm_100a (no JIT, no torch extension).

Flags: -O3 -lineinfo, NO fast-math, -ftz=false -prec-div=true -prec-sqrt=true
(subnormal thresholds and inputs must compare exactly).
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libbridger.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

SOURCES = ["api.cu", "traverse.cu", "trav_inst_i64.cu", "trav_inst_i64_ml.cu", "trav_inst_f64.cu",
           "trav_inst_gt_i64.cu", "trav_inst_gt_f64.cu", "trav_inst_sparse.cu", "trav_inst_hybrid.cu", "trav_inst_split.cu", "trav_inst_stream.cu", "trav_inst_stream_split.cu", "trav_inst_stream_codes.cu", "trav_deep.cu", "trav_deep_inst_0.cu", "trav_deep_inst_1.cu", "trav_deep_inst_2.cu", "trav_deep_inst_3.cu", "trav_deep_inst_4.cu", "gemm_path.cu", "linear.cu", "probe.cu", "lowering.cpp"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-ftz=false", "-prec-div=true", "-prec-sqrt=true",
          "-fmad=true", "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off",
          "-I", os.path.join(HERE, "..", "include")]


def _newest_src_mtime() -> float:
    t = 0.0
    for root in (CSRC, os.path.join(HERE, "..", "include")):
        for f in os.listdir(root):
            t = max(t, os.path.getmtime(os.path.join(root, f)))
    return max(t, os.path.getmtime(__file__))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= _newest_src_mtime():
        return LIB
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    # headers are shared by most units: a newer header rebuilds everything,
    # otherwise only the units whose own source changed (incremental build)
    hdr_t = max([os.path.getmtime(os.path.join(CSRC, f)) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))] +
                [os.path.getmtime(os.path.join(HERE, "..", "include", f))
                 for f in os.listdir(os.path.join(HERE, "..", "include"))] + [os.path.getmtime(__file__)])
    objs, cmds = [], []
    for s in SOURCES:
        src = os.path.join(CSRC, s)
        obj = os.path.join(objdir, s + ".o")
        objs_ok = os.path.exists(obj) and os.path.getmtime(obj) >= max(hdr_t, os.path.getmtime(src))
        if objs_ok and not force:
            objs.append(obj)
            continue
        cmd = [NVCC, *ARCH, *COMMON, "-c", src, "-o", obj]
        if s.endswith(".cu"):
            cmd += ["-Xptxas", "-v"] if verbose else []
        else:
            cmd = ["g++", "-O3", "-std=c++17", "-fPIC", "-ffp-contract=off",
                   "-I", os.path.join(HERE, "..", "include"), "-c", src, "-o", obj]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        cmds.append(cmd)
        objs.append(obj)
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=max(1, min(len(cmds), os.cpu_count() or 4))) as ex:
        for r in ex.map(lambda c: subprocess.run(c).returncode, cmds):
            if r != 0:
                raise subprocess.CalledProcessError(r, "nvcc")
    cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-cudart", "static"]
    subprocess.check_call(cmd)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)

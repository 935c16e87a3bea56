#!/usr/bin/env python
"""Linear models on the device (bridger_linear_*): throughput
and HBM roofline of the one streaming kernel (linear.cu), one JSON line per
workload.

The kernel reads X once (N*F*4 B) and writes the result (labels 4 B/row or
K fp32 scores); it is HBM-bound, so the roofline is algorithmic bytes
(X + output) / CUDA-event kernel time against MEASURED_PEAKS.json hbm_gbs.
Workloads reuse the tree configs' X shapes (C2: 1M x 28 binary logistic
regression; C3: 10M x 90 linear regression; C4-shaped: 8M x 64, 8-class
softmax behind a StandardScaler).  Same timing rules as bench.py: >= 3
warm-ups, L2 flushed (256 MiB write) before every timed step outside the
events, CUDA events on the launching stream.

  python tools/bench_linear.py [--steps K --warmup W]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
from types import SimpleNamespace

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

WORKLOADS = [
    # name, rows, F, K, task, post, scaler
    ("LR-C2shape binary logistic regression", 1_000_000, 28, 1, 1, 1, False),
    ("LinReg-C3shape regression", 10_000_000, 90, 1, 0, 0, False),
    ("Softmax-C4shape 8-class + StandardScaler", 8_000_000, 64, 8, 1, 2, True),
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--only", default=None, help="run the workloads whose name contains this string")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    import torch

    import paper_2405_12491_b200 as B
    from synth import gen_x_torch

    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
        pk = json.load(fh)
    hbm = next((pk[k] for k in ("hbm_gbs", "hbm_copy_gbs", "hbm_GBps") if k in pk), 7700.0)
    dev = torch.device("cuda", 0)
    st = torch.cuda.current_stream(dev)
    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
    for name, n, F, K, task, post, scaler in WORKLOADS:
        if args.only and args.only not in name:
            continue
        rng = np.random.default_rng(7)
        m = SimpleNamespace(n_features=F, n_outputs=K, coef=rng.normal(size=(K, F)) * 0.3,
                            intercept=rng.normal(size=K) * 0.1,
                            mean=rng.normal(size=F) if scaler else None,
                            scale=rng.uniform(0.5, 2.0, size=F) if scaler else None, task=task, post=post)
        g = B.LinearModel(m)
        X = gen_x_torch(11, 0, n, F, device=dev)
        out = (torch.empty(n, dtype=torch.int32, device=dev) if task == 1
               else torch.empty((n, K), dtype=torch.float32, device=dev))
        for _ in range(args.warmup):
            flush.fill_(1.0)
            g.predict(X, out=out)
        torch.cuda.synchronize(dev)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        l0 = B.launch_count()
        for e0, e1 in ev:
            flush.fill_(1.0)
            e0.record(st)
            g.predict(X, out=out)
            e1.record(st)
        torch.cuda.synchronize(dev)
        launches = B.launch_count() - l0
        ms = sum(a.elapsed_time(b) for a, b in ev) / args.steps
        alg = n * F * 4 + out.numel() * out.element_size()
        ach = alg / (ms / 1e3) / 1e9
        print(json.dumps({
            "metric": "linear-model inference rows/sec", "value": n / (ms / 1e3), "unit": "rows/s", "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "dtype": "f64 dot (feature order, no FMA)", "data": "synthetic",
            "config": {"workload": name, "n_rows": n, "n_features": F, "n_outputs": K,
                       "l2": "flushed before every timed step (256 MiB write)"},
            "gpu_launches": launches,
            "roofline": {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                         "traffic": None, "kernel": "linear kernel (linear.cu)",
                         "alg_bytes_per_launch": alg}}), flush=True)
        g.close()
        del X, out


if __name__ == "__main__":
    main()

"""Kernel exploration on a GPU box: time one workload's predict (CUDA events,
L2 flushed, W warm-ups) under the current BRIDGER_* environment and print one
JSON line with the step time and the library-measured dominant-kernel time.

  python tools/explore.py C5 --rows 1000000 --trees 1250 [--steps 5] [--proba] [--variant traverse]

Used with tools/gpu.sh; not part of the product or the bench contract."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2405_12491_b200 as B  # noqa: E402
from synth import gen_x_torch, make_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("config")
ap.add_argument("--rows", type=int, default=None)
ap.add_argument("--trees", type=int, default=None)
ap.add_argument("--steps", type=int, default=5)
ap.add_argument("--warmup", type=int, default=2)
ap.add_argument("--proba", action="store_true")
ap.add_argument("--variant", default=None)
ap.add_argument("--tag", default="")
ap.add_argument("--no-hot", action="store_true", help="no per-kernel events (lets programmatic dependent launch overlap)")
a = ap.parse_args()
cfg, m = make_config(a.config, n_trees=a.trees)
n = a.rows or cfg.n_rows
X = gen_x_torch(cfg.seed, 0, n, cfg.n_features, device="cuda")
g = B.Model(m, device=0, variant=a.variant)
flush = torch.empty(64 << 20, device="cuda")
if a.proba:
    out = torch.empty((n, max(2, cfg.n_classes)), device="cuda")
    call = lambda: g.predict_proba(X, out=out)
else:
    out = (torch.empty(n, dtype=torch.int32, device="cuda") if cfg.kind == "classification"
           else torch.empty((n, cfg.n_classes), device="cuda"))
    call = lambda: g.predict(X, out=out)
for _ in range(a.warmup):
    flush.fill_(1.0)
    call()
torch.cuda.synchronize()
B.hot_kernel_timing(not a.no_hot)
for k in range(4):
    B.hot_kernel_time(k)
tot = 0.0
for _ in range(a.steps):
    flush.fill_(1.0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    call()
    e1.record()
    torch.cuda.synchronize()
    tot += e0.elapsed_time(e1)
hot = [B.hot_kernel_time(k) for k in range(4)]
B.hot_kernel_timing(False)
env = {k: v for k, v in os.environ.items() if k.startswith("BRIDGER_")}
print(json.dumps({"tag": a.tag, "config": a.config, "rows": n, "trees": m.n_trees, "env": env,
                  "ms_per_step": tot / a.steps, "rows_per_s": n / (tot / a.steps / 1e3),
                  "hot_ms": [h[0] / max(1, h[1]) for h in hot], "hot_launches": [h[1] for h in hot],
                  "layout": g.layout(), "info": g.info()}), flush=True)

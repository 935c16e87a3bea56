"""Measure the per-depth variant table that AUTO variant selection follows
(BASELINE.json north star: "the variant is chosen per tree depth from measured
throughput"; SPEC.md:340 frames the same choice: gather loop vs matrix form).

For D = 1..12: a C2-shaped random forest (100 trees of depth D, 28 features,
binary classification), 1M rows, L2 flushed, CUDA events, median of 5:
traversal (K4/K4d, threshold-bin codes where the lowering picks them) vs the
fused GEMM form K5 (variant gemm) vs staged K1 -> K2 -> K3 (gemm_staged), the
latter two for D <= 8 only (the path matrix C_D outgrows one SM beyond).
Writes profiles/variant_table.json; tools/gen_variant_table.py turns it into
paper_2405_12491_b200/csrc/variant_table.h, which bridger's AUTO reads."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2405_12491_b200 as B  # noqa: E402
from synth import gen_x_torch, perfect_ensemble  # noqa: E402

N, T, F = 1_000_000, 100, 28
X = gen_x_torch(2, 0, N, F, device="cuda")
flush = torch.empty(64 << 20, device="cuda")
out = torch.empty(N, dtype=torch.int32, device="cuda")
rows = []
for D in range(1, 13):
    m = perfect_ensemble(100 + D, T, D, F, kind="classification", n_classes=2, calib_rows=2048)
    rec = {"depth": D, "n_trees": T, "rows": N, "features": F}
    for v in ("traverse", "gemm", "gemm_staged", "gemm_sparse"):
        if v != "traverse" and D > 8:
            continue
        g = B.Model(m, device=0, variant=v)
        ts = []
        for it in range(7):
            flush.fill_(1.0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.predict(X, out=out)
            e1.record()
            torch.cuda.synchronize()
            if it >= 2:
                ts.append(e0.elapsed_time(e1))
        rec[v + "_ms"] = statistics.median(ts)
        if v == "traverse":
            rec["traverse_format"] = g.layout()["format"]
        g.close()
    best = min((k for k in rec if k.endswith("_ms")), key=lambda k: rec[k])
    rec["best"] = best[:-3]
    rows.append(rec)
    print(json.dumps(rec), flush=True)
os.makedirs("profiles", exist_ok=True)
json.dump({"gpu": torch.cuda.get_device_name(), "how": __doc__.strip().splitlines()[0], "rows": rows},
          open("profiles/variant_table.json", "w"), indent=1)

#!/usr/bin/env python
"""Tree-ensemble inference benchmark (BASELINE.json metric: rows/s at 1/2/4/8 B200).

One step = one pass of the whole hot path (lowering is done
once at load; per step: feature gather + compare / traversal, leaf-value gather,
per-tree reduction, finalize) over one batch of synthetic rows.  Default
workload = BASELINE.json configs[1] (C2: random forest, 100 trees, depth 8,
1M rows x 28 features, binary classification; predict -> int32 labels).

  python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--config C2]
  python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N   (row shards, weak scaling)

Timing: W untimed warm-ups, then K steps each bracketed by CUDA events on the
launching stream; L2 is flushed (256 MiB write) before every step, outside the
events; barrier + synchronize on both sides of the timed region; max over
ranks.  `e2e` re-times the same metric through the public host-buffer API
(bridger_predict_host: H2D of the pinned input + predict + D2H of the labels
inside the timed region).  `roofline` reports the dominant kernel (traversal)
against the shared-memory pipe, its binding resource.
`cpu_baseline` is the oracle (oracle/) timed on this host's cores on a bounded
sample (a reported baseline, not the target).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms", "100",
                 "-i", str(self.index)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                out = ""
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm, mx, reasons = [], None, set()
        for l in getattr(self, "lines", []):
            p = [x.strip() for x in l.split(",")]
            if len(p) < 6:
                continue
            try:
                sm.append(float(p[0]))
                mx = float(p[1])
            except ValueError:
                continue
            for n, v in zip(names, p[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def cpu_baseline(m, cfg, target_s=10.0):
    """The oracle as it stands, on this host's cores, on a bounded row sample."""
    import oracle
    from synth import gen_x
    cores = oracle.n_cores()
    n = 4096
    X = gen_x(cfg.seed, 0, n, cfg.n_features)
    t = time.perf_counter()
    oracle.run(m, X, n_threads=cores, want=("label", "pred"))
    dt = time.perf_counter() - t
    n2 = int(min(cfg.n_rows, max(n, n * (target_s * 0.8) / max(dt, 1e-6))))
    X = gen_x(cfg.seed, 0, n2, cfg.n_features)
    t = time.perf_counter()
    oracle.run(m, X, n_threads=cores, want=("label", "pred"))
    dt = time.perf_counter() - t
    return {"value": n2 / dt, "unit": "rows/s", "cores": cores, "kind": "oracle",
            "sample": f"rows [0, {n2}) of the {cfg.name} input ({n2}/{cfg.n_rows} rows), all {cfg.n_trees} trees, "
                      f"{dt:.1f} s"}


def run_reference(args):
    """--impl reference: the oracle timed on host cores, same metric/config."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    import oracle
    from synth import gen_x, make_config
    cfg, m = make_config(args.config)
    cores = oracle.n_cores()
    # per step: a bounded sample sized so warmup+steps finish in ~2 minutes
    probe = gen_x(cfg.seed, 0, 2048, cfg.n_features)
    t = time.perf_counter()
    oracle.run(m, probe, n_threads=cores, want=("label", "pred"))
    rate = 2048 / (time.perf_counter() - t)
    per_step_s = min(8.0, 120.0 / max(1, args.steps + args.warmup))
    n = int(max(2048, min(cfg.n_rows, rate * per_step_s)))
    X = gen_x(cfg.seed, 0, n, cfg.n_features)
    for _ in range(args.warmup):
        oracle.run(m, X[: min(n, 4096)], n_threads=cores, want=("label", "pred"))
    times = []
    for _ in range(args.steps):
        t = time.perf_counter()
        oracle.run(m, X, n_threads=cores, want=("label", "pred"))
        times.append(time.perf_counter() - t)
    tot = sum(times)
    value = n * args.steps / tot
    line = {
        "impl": "reference", "metric": "tree-ensemble inference rows/sec", "value": value, "unit": "rows/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32 compare, f64 accumulate",
        "data": "synthetic", "config": workload_config(cfg, world),
        "cpu_baseline": {"value": value, "unit": "rows/s", "cores": cores, "kind": "oracle",
                         "sample": f"{n} rows per step (bounded sample of the {cfg.n_rows}-row workload)"},
        "e2e": {"value": value, "unit": "rows/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def gemm_roofline(B, m, cfg, X, dev, args):
    """The paper's GEMM form of steps a1..a4 on the same input (the variant AUTO
    does not pick), in both pipelines:
    * fused K5 (variant "gemm"): one warp-specialised kernel,
      decisions only in shared memory; int8 tcgen05 throughput of the whole
      kernel vs the measured int8 tensor peak;
    * staged K1 -> K2 -> K3 (variant "gemm_staged"): the K2 path-contraction
      kernel alone vs the int8 peak, K1 vs HBM."""
    import torch
    try:
        with open(os.path.join(ROOT, "profiles", "int8_peak.json")) as fh:
            peak = json.load(fh)["int8_tops_burst"]
            src = "measured (profiles/int8_peak.json: cuBLASLt s8 8192^3)"
    except Exception:
        peak, src = 2 * _peaks()[0].get("bf16_tflops", 1590.0), "bf16 measured x 2 (nominal int8/bf16 ratio)"
    n = X.shape[0]
    out = torch.empty(n, dtype=torch.int32, device=dev) if cfg.kind == "classification" else torch.empty((n, 1), device=dev)
    ip, lp = B.gemm_geometry(cfg.depth)
    steps = 2

    def timed(variant):
        g = B.Model(m, device=dev.index, variant=variant)
        for _ in range(2):
            g.predict(X, out=out)
        torch.cuda.synchronize(dev)
        B.hot_kernel_timing(True)
        for k in range(4):
            B.hot_kernel_time(k)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            g.predict(X, out=out)
        e1.record()
        torch.cuda.synchronize(dev)
        ks = [B.hot_kernel_time(k) for k in range(4)]
        B.hot_kernel_timing(False)
        g.close()
        return e0.elapsed_time(e1) / steps, ks

    ops = 2.0 * n * cfg.n_trees * ip * lp * steps        # dense int8 ops of the contraction (padded)
    f_ms, fk = timed("gemm")
    k5_ms, k5_n = fk[3]
    fused = {"kernel": "fz_kernel (K5: producer warps -> SMEM decisions -> tcgen05.mma kind::i8 -> TMEM -> "
                       "leaf select/gather/reduce epilogue)", "bound": "tensor",
             "achieved": ops / (k5_ms / 1e3) / 1e12, "peak": peak, "unit": "TOP/s",
             "frac": ops / (k5_ms / 1e3) / 1e12 / peak, "peak_source": src,
             "k5_ms_per_step": k5_ms / steps, "k5_launches_per_step": k5_n // steps,
             "decisions_per_s": n * cfg.n_trees * ((1 << cfg.depth) - 1) * steps / (k5_ms / 1e3),
             "ms_per_step": f_ms, "rows_per_s": n / (f_ms / 1e3)}
    s_ms, sk = timed("gemm_staged")
    k2_ms, k2_n = sk[0]
    k1_ms, k3_ms = sk[1][0], sk[2][0]
    k1_bytes = steps * (n * cfg.n_features * 4 + n * cfg.n_trees * ip)
    hbm = _peaks()[0].get("hbm_gbs", 6541.1)
    gather = {"kernel": "gc_kernel (a1+a2: exact fp32 gather + less_equal, int8 decisions)", "bound": "hbm",
              "achieved": k1_bytes / (k1_ms / 1e3) / 1e9, "peak": hbm, "unit": "GB/s",
              "frac": k1_bytes / (k1_ms / 1e3) / 1e9 / hbm, "ms_per_step": k1_ms / steps,
              "k3_leaf_gather_ms_per_step": k3_ms / steps}
    achieved = ops / (k2_ms / 1e3) / 1e12
    return {"kernel": "pc_kernel (tcgen05.mma.cta_group::1.kind::i8, TMEM accumulators)", "bound": "tensor",
            "achieved": achieved, "peak": peak, "unit": "TOP/s", "frac": achieved / peak, "peak_source": src,
            "k2_ms_per_step": k2_ms / steps, "k2_launches_per_step": k2_n // steps,
            "gemm_variant_ms_per_step": s_ms, "gemm_variant_rows_per_s": n / (s_ms / 1e3),
            "gather_compare": gather, "fused": fused,
            "note": "GEMM form of a1..a4: 'fused' = K5 (variant gemm), the rest = staged K1->K2->K3 "
                    "(variant gemm_staged); AUTO selects the traversal"}


def workload_config(cfg, world):
    return {"workload": f"{cfg.name}: {cfg.describe}", "n_rows_per_gpu": cfg.n_rows, "n_trees": cfg.n_trees,
            "depth": cfg.depth, "n_features": cfg.n_features, "n_outputs": cfg.n_classes,
            "sharding": (f"{cfg.sharding} x{world}" if world > 1 else "single GPU"),
            "l2": "flushed before every timed step (256 MiB write)", "output": "predict (int32 labels)"
            if cfg.kind == "classification" else "predict (fp32 scores)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2")
    ap.add_argument("--variant", default=None, choices=[None, "auto", "traverse", "gemm", "gemm_staged"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-gemm", action="store_true", help="skip the GEMM-form (tcgen05) sub-measurement")
    ap.add_argument("--e2e-steps", type=int, default=7)
    ap.add_argument("--rows", type=int, default=None, help="override rows per GPU (exploration; reported in config)")
    ap.add_argument("--trees", type=int, default=None, help="override ensemble size (exploration)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    import paper_2405_12491_b200 as B
    from synth import gen_x, gen_x_torch, make_config

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        # bind the process group to this rank's GPU before the first collective
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    cfg, m = make_config(args.config, n_trees=args.trees)
    if args.rows or args.trees:
        import dataclasses
        cfg = dataclasses.replace(cfg, n_rows=args.rows or cfg.n_rows, n_trees=m.n_trees,
                                  describe=cfg.describe + f" [override: {args.rows or cfg.n_rows} rows, {m.n_trees} trees]")
    n = cfg.n_rows
    tree_sharded = cfg.sharding == "trees"
    # row sharding: each rank its own rows (weak scaling); tree sharding: all
    # rows on every rank, trees split, one NCCL reduce-scatter (strong scaling)
    row0 = 0 if tree_sharded else rank * n
    X = gen_x_torch(cfg.seed, row0, n, cfg.n_features, device=dev)
    tsp = None
    if tree_sharded and world > 1:
        from paper_2405_12491_b200.dist import TreeShardedPredictor
        tsp = TreeShardedPredictor(m, device=local)
        model = tsp.model
    else:
        model = B.Model(m, device=local, variant=args.variant)
    classif = cfg.kind == "classification"
    out = torch.empty(n, dtype=torch.int32, device=dev) if classif else torch.empty((n, 1), device=dev)
    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)  # 256 MiB > 126 MB L2
    st = torch.cuda.current_stream(dev)

    def step():
        if tsp is not None:
            return tsp.predict(X)
        return model.predict(X, out=out)

    for _ in range(args.warmup):
        flush.fill_(1.0)
        step()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    B.hot_kernel_timing(True)
    B.hot_kernel_time()
    l0 = B.launch_count()
    with ClockSampler(local) as clk:
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        t_wall = time.perf_counter()
        for e0, e1 in ev:
            flush.fill_(1.0)
            e0.record(st)
            step()
            e1.record(st)
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        t_wall = time.perf_counter() - t_wall
    launches = B.launch_count() - l0
    hot_ms, hot_n = B.hot_kernel_time()
    if hot_n == 0:  # fused GEMM-form variant: its one kernel is K5
        hot_ms, hot_n = B.hot_kernel_time(3)
    B.hot_kernel_timing(False)
    step_ms = sum(e0.elapsed_time(e1) for e0, e1 in ev)
    t = torch.tensor([step_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_per_step = t.item() / args.steps
    value = (n if tree_sharded else n * world) / (ms_per_step / 1e3)

    # ---- e2e through the public host-buffer API (pinned input, labels back to host)
    if tsp is not None:
        args.e2e_steps = 0  # the host-buffer API runs a whole model on one device
    Xh = (torch.from_numpy(gen_x(cfg.seed, row0, n, cfg.n_features)) if args.e2e_steps > 0
          else torch.zeros((32, cfg.n_features))).pin_memory()
    oh = torch.empty(n, dtype=torch.int32).pin_memory() if classif else torch.empty((n, 1)).pin_memory()
    if args.e2e_steps > 0:
        model.predict_host(Xh, out=oh)
    e2e_times = []
    for _ in range(args.e2e_steps):
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        model.predict_host(Xh, out=oh)
        e2e_times.append(time.perf_counter() - t0)
    # median over the e2e steps: host-side timing on a shared box is noisy (one
    # slow step would dominate a mean)
    te = torch.tensor([statistics.median(e2e_times) if e2e_times else 0.0], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e = {"value": (n if tree_sharded else n * world) / te.item() if e2e_times else None, "unit": "rows/s", "h2d_bytes_per_step": n * cfg.n_features * 4,
           "d2h_bytes_per_step": int(oh.numel() * oh.element_size()),
           "api": "bridger_predict_host (2-stream chunked H2D/compute/D2H pipeline)"}

    # ---- roofline of the dominant kernel
    peaks, src = _peaks()
    info = model.info()
    clocks = clk.summary()
    variant = info["variant"]
    hot_avg = hot_ms / max(1, hot_n)
    if variant == "traverse":
        # algorithmic shared-memory bytes per launch, per (row, tree): D node records +
        # D feature values + K leaf values, each per-lane access counted in whole
        # 32-bit bank words (a warp-wide access of b < 4 bytes per lane still
        # occupies one 128-byte wavefront): fp32 nodes 8 B + x 4 B -> 12 D + 4 K;
        # threshold-bin codes 4 B nodes + u16 codes -> 8 D + 4 K
        coded = model.layout().get("coded", False)
        alg = n * model.n_trees * ((8 if coded else 12) * cfg.depth + 4 * cfg.n_classes)
        sm_count = torch.cuda.get_device_properties(dev).multi_processor_count
        peak = sm_count * 128 * peaks.get("sm_max_mhz", 1965.0) * 1e6 / 1e9   # GB/s, guide unit counts
        psrc = f"derived from guide unit counts ({src} sm_max_mhz)"
        try:  # measured on this pool's B200 by tools/smem_peak.cu (conflict-free LDS.64)
            with open(os.path.join(ROOT, "profiles", "smem_peak.json")) as fh:
                peak = json.load(fh)["smem_lds64_conflict_free_GBps"]
                psrc = "measured (profiles/smem_peak.json: tools/smem_peak.cu, conflict-free LDS.64)"
        except Exception:
            pass
        achieved = alg / (hot_avg / 1e3) / 1e9
        roof = {"bound": "alu", "resource": "shared-memory (LSU) pipe bandwidth",
                "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak, "traffic": None,
                "kernel": "trav_kernel", "kernel_ms": hot_avg,
                "node_format": ("threshold-bin codes (4 B nodes, u16 inputs; bin_kernel pass)" if coded
                                else "tree-streamed, fp32 thresholds" if model.layout().get("format") == "stream"
                                else "fp32 (8 B nodes)"),
                "visits_per_s": n * model.n_trees * cfg.depth / (hot_avg / 1e3),
                "hbm_frac": (n * cfg.n_features * 4 + n * 4) / (hot_avg / 1e3) / 1e9 / peaks["hbm_gbs"],
                "peak_source": psrc}
    else:
        ip, lp = B.gemm_geometry(cfg.depth)
        try:
            with open(os.path.join(ROOT, "profiles", "int8_peak.json")) as fh:
                ipeak = json.load(fh)["int8_tops_burst"]
        except Exception:
            ipeak = 2 * peaks.get("bf16_tflops", 1590.0)
        ach = 2.0 * n * model.n_trees * ip * lp / (hot_avg / 1e3) / 1e12 if hot_avg > 0 else None
        roof = {"bound": "tensor", "achieved": ach, "peak": ipeak, "unit": "TOP/s",
                "frac": ach / ipeak if ach else None, "traffic": None,
                "kernel": "fz_kernel" if variant == "gemm" else "pc_kernel", "kernel_ms": hot_avg}
    tr = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tr):
        try:
            roof["traffic"] = json.load(open(tr)).get(f"{cfg.name}:{variant}")
        except Exception:
            pass

    line = {
        "metric": "tree-ensemble inference rows/sec", "value": value, "unit": "rows/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong" if tree_sharded else "weak", "vs_baseline": None,
        "dtype": "f32 compare, int64 fixed-point accumulate" if info["acc_is_int64"] else "f32 compare, f64 accumulate",
        "data": "synthetic (counter-based generator, seeded; random calibrated trees)",
        "config": workload_config(cfg, world), "variant": variant, "exact_tier": info["exact_tier"],
        "gpu_launches": launches, "wall_s_timed": t_wall, "roofline": roof, "e2e": e2e, "clocks": clocks,
    }
    if cfg.depth <= 8 and not args.no_gemm:
        line["path_contraction"] = gemm_roofline(B, m, cfg, X, dev, args)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(m, cfg)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

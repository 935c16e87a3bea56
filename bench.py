#!/usr/bin/env python
"""Tree-ensemble inference benchmark (BASELINE.json metric: rows/s at 1/2/4/8
B200, with % of the binding roofline per kernel).

One step = one pass of the whole hot path (lowering is done
once at load; per step: threshold-bin coding of the input / feature gather +
compare / traversal, leaf-value gather, per-tree reduction, finalize) over one
batch of synthetic rows.  Default workload = the largest single-GPU config of
BASELINE.json `configs` (C3: gradient-boosted trees, 500 trees, depth 6,
10M rows x 90 features, regression -> fp32 scores); C4/C5 are the configs
BASELINE.json marks as sharded over 8 GPUs.

  python bench.py [--gpus N --steps K --warmup W] [--config C3] [--impl reference]
  python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N

`--gpus N` without a torchrun environment re-launches itself through
torch.distributed.run with N ranks (one per GPU, NCCL).  Row-sharded configs
(C1..C4) split the config's TOTAL rows into contiguous shards (strong scaling:
the job is the config's N rows whatever the GPU count; no data-path
collective); C5 is tree-sharded (every rank all rows, a contiguous share of the
trees, ONE NCCL int64 reduce-scatter).

Timing: W >= 3 untimed warm-ups, then K steps each bracketed by CUDA events on
the launching stream; L2 is flushed (256 MiB write) before every step, outside
the events; barrier + synchronize on both sides of the timed region; max over
ranks; nvidia-smi clocks sampled during the timed region.  `e2e` re-times the
same metric through the public host-buffer API (pinned host rows -> H2D ->
predict -> D2H of the outputs, all inside the timed region).  `roofline`
reports the dominant kernel against the shared-memory (LSU) pipe bandwidth
measured live on this GPU (bridger_probe_smem_bandwidth), its binding
resource.  `cpu_baseline` is the oracle (oracle/) timed on this
host's cores on a bounded sample (a reported baseline, not the target).
At N=1 the line also carries `extra`: the C2 workload, the C4 forest on 1M
rows and a 1250-tree C5 shard (the per-GPU slice at 8 GPUs) on 1M rows, each
with its own roofline (predict_proba timed too for the classifiers).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "tree-ensemble inference rows/sec"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms", "100",
                 "-i", str(self.index)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
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
        for l in self.lines:
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


def row_range(n_rows: int, world: int, rank: int):
    """Contiguous row shard [a, b) of rank (the same rule as dist.row_range)."""
    per = -(-n_rows // world)
    a = min(n_rows, rank * per)
    return a, min(n_rows, a + per)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def relaunch(args_list, n):
    """--gpus N outside torchrun: start N ranks through torch.distributed.run
    (one process per GPU, rendezvous on 127.0.0.1) and return its exit code."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__), *args_list]
    env = dict(os.environ, OMP_NUM_THREADS=os.environ.get("OMP_NUM_THREADS", "1"))
    return subprocess.call(cmd, env=env)


# --------------------------------------------------------------- cpu leg ----
def cpu_baseline(m, cfg, budget_s=12.0):
    """The oracle as it stands on this host's cores: a bounded sample of the
    workload's rows, best of 3 on all cores, plus one single-core run."""
    import oracle
    from synth import gen_x
    cores = oracle.n_cores()
    probe = 1024
    X = gen_x(cfg.seed, 0, probe, cfg.n_features)
    t = time.perf_counter()
    oracle.run(m, X, n_threads=cores, want=("label", "pred"))
    rate = probe / max(time.perf_counter() - t, 1e-6)
    n = int(min(cfg.n_rows, max(probe, rate * budget_s / 4)))
    X = gen_x(cfg.seed, 0, n, cfg.n_features)
    best = 1e30
    for _ in range(3):
        t = time.perf_counter()
        oracle.run(m, X, n_threads=cores, want=("label", "pred"))
        best = min(best, time.perf_counter() - t)
    n1 = int(max(256, min(n, rate / cores * budget_s / 6)))
    t = time.perf_counter()
    oracle.run(m, X[:n1], n_threads=1, want=("label", "pred"))
    one = n1 / (time.perf_counter() - t)
    return {"value": n / best, "unit": "rows/s", "cores": cores, "kind": "oracle",
            "single_core_rows_per_s": one,
            "sample": f"rows [0, {n}) of the {cfg.name} input ({n}/{cfg.n_rows} rows), all {cfg.n_trees} trees, "
                      f"best of 3 on {cores} threads ({best:.2f} s); single core on {n1} rows"}


def run_reference(args):
    """--impl reference: the oracle timed on host cores, same metric/config.
    Under torchrun only rank 0 runs it; the other ranks exit without work."""
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    import oracle
    from synth import gen_x, make_config
    cfg, m = make_config(args.config)
    cores = oracle.n_cores()
    # per step: a bounded sample sized so warmup + steps finish in ~2 minutes
    probe = gen_x(cfg.seed, 0, 1024, cfg.n_features)
    t = time.perf_counter()
    oracle.run(m, probe, n_threads=cores, want=("label", "pred"))
    rate = 1024 / (time.perf_counter() - t)
    per_step_s = min(8.0, 120.0 / max(1, args.steps + args.warmup))
    n = int(max(1024, min(cfg.n_rows, rate * per_step_s)))
    X = gen_x(cfg.seed, 0, n, cfg.n_features)
    for _ in range(args.warmup):
        oracle.run(m, X[: min(n, 1024)], n_threads=cores, want=("label", "pred"))
    times = []
    for _ in range(args.steps):
        t = time.perf_counter()
        oracle.run(m, X, n_threads=cores, want=("label", "pred"))
        times.append(time.perf_counter() - t)
    tot = sum(times)
    value = n * args.steps / tot
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "rows/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32 compare, f64 accumulate", "data": "synthetic", "config": workload_config(cfg, 1),
        "cpu_baseline": {"value": value, "unit": "rows/s", "cores": cores, "kind": "oracle",
                         "sample": f"{n} rows per step (bounded sample of the {cfg.n_rows}-row workload)"},
        "e2e": {"value": value, "unit": "rows/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------ roofline ----
_SMEM_PEAK = {}


def smem_peak(B, dev_index):
    """Shared-memory pipe peak measured live on this GPU (conflict-free LDS.64)."""
    if dev_index not in _SMEM_PEAK:
        cf, rnd = B.probe_smem_bandwidth(dev_index)
        _SMEM_PEAK[dev_index] = (cf, rnd)
    return _SMEM_PEAK[dev_index]


def int8_peak(dev):
    """Dense int8 tensor peak measured live: cuBLASLt s8 x s8 -> s32 8192^3
    (torch._int_mm), best of 5 -- the denominator for the path contraction."""
    import torch
    n = 8192
    a = torch.randint(-2, 2, (n, n), dtype=torch.int8, device=dev)
    b = torch.randint(-2, 2, (n, n), dtype=torch.int8, device=dev).t().contiguous().t()
    for _ in range(2):
        torch._int_mm(a, b)
    torch.cuda.synchronize(dev)
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch._int_mm(a, b)
        e1.record()
        torch.cuda.synchronize(dev)
        best = min(best, e0.elapsed_time(e1) / 1e3)
    del a, b
    return 2 * n ** 3 / best / 1e12


def trav_roofline(B, model, cfg, n, hot_avg_ms, dev_index, n_trees=None):
    """Dominant traversal kernel vs the shared-memory (LSU) pipe: algorithmic
    bytes per (row, tree) = D node records + D input values + K leaf values,
    each per-lane access counted in whole 32-bit bank words (a warp access of
    b < 4 bytes per lane still takes a full 128-byte wavefront): fp32 nodes
    8 B + x 4 B -> 12 D + 4 K; threshold-bin codes 4 B nodes + u16 codes ->
    8 D + 4 K  (DESIGN.md §6 "Roofline")."""
    peaks, psrc = _peaks()
    lay = model.layout()
    coded = lay.get("coded", False)
    T = model.n_trees if n_trees is None else n_trees
    per = (8 if coded else 12) * cfg.depth + 4 * cfg.n_classes
    alg = n * T * per
    cf, rnd = smem_peak(B, dev_index)
    achieved = alg / (hot_avg_ms / 1e3) / 1e9
    kern = ("trav_stream_kernel" if lay["format"].startswith("stream") else
            "trav_deep_kernel" if lay["format"] == "codes_deep" else "trav_kernel")
    return {"bound": "alu", "resource": "shared-memory (LSU) pipe bandwidth", "kernel": kern,
            "achieved": achieved, "peak": cf, "unit": "GB/s", "frac": achieved / cf, "traffic": None,
            "kernel_ms": hot_avg_ms, "alg_bytes_per_row_tree": per, "alg_bytes_per_launch": alg,
            "node_format": lay["format"], "n_chunks": lay["n_chunks"],
            "visits_per_s": n * T * cfg.depth / (hot_avg_ms / 1e3),
            "hbm_frac": (n * cfg.n_features * 4 + n * 4) / (hot_avg_ms / 1e3) / 1e9 / peaks["hbm_gbs"],
            "peak_source": "measured live on this GPU: bridger_probe_smem_bandwidth (1 CTA x 512 threads per SM, "
                           "conflict-free LDS.64, best of 5)",
            "peak_random_lds64_gbps": rnd}


def gemm_roofline(B, m, cfg, X, dev, n_max=2_000_000):
    """The paper's GEMM form of steps a1..a4 on
    the first n_max rows of the same input (the variant AUTO does not pick):
    * fused K5 (variant "gemm"): one warp-specialised kernel, decisions only in
      shared memory; int8 tcgen05 throughput of the whole kernel vs the int8
      peak measured live;
    * staged K1 -> K2 -> K3 (variant "gemm_staged"): the K2 path-contraction
      kernel alone vs the int8 peak, K1 vs HBM."""
    import torch
    X = X[: min(X.shape[0], n_max)]
    n = X.shape[0]
    peak = int8_peak(dev)
    src = "measured live: torch._int_mm (cuBLASLt s8 8192^3), best of 5"
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
    # K2 streams every (tree, 128-row) decision tile (i_pad bytes per row-tree)
    # from HBM once: its other roofline -- the binding one at small depths
    # (C3: 64-byte rows, 64x64 contractions)
    k2_bytes = steps * n * cfg.n_trees * ip
    k2_hbm = {"bound": "hbm", "achieved": k2_bytes / (k2_ms / 1e3) / 1e9, "peak": hbm, "unit": "GB/s",
              "frac": k2_bytes / (k2_ms / 1e3) / 1e9 / hbm,
              "note": "decision tiles read once per contraction (the int8 frac above is low by construction when "
                      "each 64-byte decision row feeds only 2*64*64 ops)"}
    return {"kernel": "pc_kernel (tcgen05.mma kind::i8, TMEM accumulators)", "bound": "tensor",
            "achieved": achieved, "peak": peak, "unit": "TOP/s", "frac": achieved / peak, "peak_source": src,
            "decision_stream": k2_hbm,
            "rows": n, "k2_ms_per_step": k2_ms / steps, "k2_launches_per_step": k2_n // steps,
            "gemm_variant_ms_per_step": s_ms, "gemm_variant_rows_per_s": n / (s_ms / 1e3),
            "gather_compare": gather, "fused": fused,
            "note": f"GEMM form of a1..a4 on rows [0, {n}): 'fused' = K5 (variant gemm), the rest = staged "
                    "K1->K2->K3 (variant gemm_staged); AUTO selects per depth from the measured variant table"}


def workload_config(cfg, world, n_rows=None):
    n_rows = cfg.n_rows if n_rows is None else n_rows
    tree_sharded = cfg.sharding == "trees"
    return {"workload": f"{cfg.name}: {cfg.describe}", "n_rows": n_rows,
            "n_rows_per_gpu": n_rows if tree_sharded else -(-n_rows // world), "n_trees": cfg.n_trees,
            "depth": cfg.depth, "n_features": cfg.n_features, "n_outputs": cfg.n_classes,
            "sharding": ("single GPU" if world == 1 else
                         f"trees x{world} (all rows per GPU, one NCCL int64 reduce-scatter)" if tree_sharded
                         else f"rows x{world} (contiguous shards of the {n_rows} rows, no collective)"),
            "l2": "flushed before every timed step (256 MiB write)",
            "output": "predict (int32 labels)" if cfg.kind == "classification" else "predict (fp32 scores)"}


# ------------------------------------------------------------ GPU leg ----
def time_steps(step, steps, warmup, dev, world, flush, st, sampler=None, hot=True):
    """W untimed warm-ups, then `steps` steps each between CUDA events on the
    launching stream (L2 flush outside the events); max over ranks.  hot:
    the library also records events around its dominant kernel (the
    roofline's launch duration) -- off for the latency-only C1 line, where the
    two extra event records would be part of what is measured."""
    import torch
    import torch.distributed as dist
    import paper_2405_12491_b200 as B
    for _ in range(warmup):
        flush.fill_(1.0)
        step()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    B.hot_kernel_timing(hot)
    for k in range(4):
        B.hot_kernel_time(k)
    l0 = B.launch_count()
    ctx = sampler if sampler is not None else _Null()
    with ctx:
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
    hot = [B.hot_kernel_time(k) for k in range(4)]
    B.hot_kernel_timing(False)
    step_ms = sum(e0.elapsed_time(e1) for e0, e1 in ev)
    t = torch.tensor([step_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.item() / steps, hot, launches, t_wall


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        pass


def run_workload(name, args, dev, world, rank, local, headline, rows=None, trees=None, proba=False):
    """Build config `name` (optionally overridden rows / trees), time predict
    (and predict_proba), e2e through the host-buffer API, and the roofline."""
    import dataclasses

    import torch
    import paper_2405_12491_b200 as B
    from synth import gen_x_torch, make_config
    cfg, m = make_config(name, n_trees=trees)
    if rows or trees:
        cfg = dataclasses.replace(cfg, n_rows=rows or cfg.n_rows, n_trees=m.n_trees,
                                  describe=cfg.describe + f" [here: {rows or cfg.n_rows} rows, {m.n_trees} trees]")
    n_total = cfg.n_rows
    tree_sharded = cfg.sharding == "trees"
    if tree_sharded:
        a, b = 0, n_total
    else:
        a, b = row_range(n_total, world, rank)
    n = b - a
    # shard generation and model load are timed separately
    # (host wall clock, device synchronised; outside the timed steps)
    torch.cuda.synchronize(dev)
    t_gen = time.perf_counter()
    if name == "C1":  # C1's 150 iris-like rows are generated on the host and copied
        from synth import iris_like_x
        X = torch.from_numpy(iris_like_x(cfg.seed)[a:b]).to(dev)
    else:
        X = gen_x_torch(cfg.seed, a, n, cfg.n_features, device=dev)
    torch.cuda.synchronize(dev)
    t_gen = time.perf_counter() - t_gen
    t_load = time.perf_counter()
    tsp = None
    reduce_desc = None
    if tree_sharded and world > 1:
        from paper_2405_12491_b200.dist import FusedTreeShardedPredictor, TreeShardedPredictor
        tsp = None
        if not args.no_fused_reduce:
            tsp = FusedTreeShardedPredictor(m, device=local, variant=args.variant)
            if not tsp.available:
                tsp = None
        if tsp is not None:
            reduce_desc = ("fused: each rank's walk adds its int64 partials straight into the owner rank's "
                           "accumulator slice over NVLink P2P (CUDA IPC, red.global.add)")
        else:
            tsp = TreeShardedPredictor(m, device=local, variant=args.variant)
            reduce_desc = "NCCL reduce-scatter of int64 partials"
        model = tsp.model
    else:
        model = B.Model(m, device=local, variant=args.variant)
    torch.cuda.synchronize(dev)
    t_load = time.perf_counter() - t_load
    classif = cfg.kind == "classification"
    out = torch.empty(n, dtype=torch.int32, device=dev) if classif else torch.empty((n, cfg.n_classes), device=dev)
    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)  # 256 MiB > 126 MB L2
    st = torch.cuda.current_stream(dev)

    def step():
        if tsp is not None:
            return tsp.predict(X)
        return model.predict(X, out=out)

    steps = args.steps if headline else max(3, min(args.steps, 8))
    clk = ClockSampler(local) if headline else None
    latency_only = name == "C1" and not headline  # the C1 extra: launch latency, no meaningful roofline
    ms, hot, launches, t_wall = time_steps(step, steps, args.warmup, dev, world, flush, st, clk, hot=not latency_only)
    res = {"value": n_total / (ms / 1e3), "ms_per_step": ms, "steps": steps, "gpu_launches": launches,
           "wall_s_timed": t_wall, "config": workload_config(cfg, world, n_total),
           "setup_s": {"input_generation": t_gen, "model_load": t_load,
                       "note": "untimed: seeded shard generation on the device; lowering + upload of the model"}}
    if reduce_desc:
        res["config"]["reduce"] = reduce_desc
    if clk is not None:
        res["clocks"] = clk.summary()
    info = model.info()
    res["variant"] = info["variant"]
    res["exact_tier"] = info["exact_tier"]
    res["dtype"] = ("f32 compare (u16 threshold-bin codes), int64 fixed-point accumulate" if info["acc_is_int64"]
                    else "f32 compare, f64 accumulate")
    hot_ms, hot_n = hot[0]
    if hot_n == 0:
        hot_ms, hot_n = hot[3]
    hot_avg = hot_ms / max(1, hot_n)
    if latency_only:
        res["roofline"] = None
    elif info["variant"] == "traverse":
        res["roofline"] = trav_roofline(B, model, cfg, n, hot_avg, local)
        res["roofline"]["kernel_share_of_step"] = hot_ms / steps / ms
    else:
        ip, lp = B.gemm_geometry(cfg.depth)
        ach = 2.0 * n * model.n_trees * ip * lp / (hot_avg / 1e3) / 1e12 if hot_avg > 0 else None
        pk = int8_peak(dev)
        res["roofline"] = {"bound": "tensor", "achieved": ach, "peak": pk, "unit": "TOP/s",
                           "frac": ach / pk if ach else None, "traffic": None,
                           "kernel": "fz_kernel" if info["variant"] == "gemm" else "pc_kernel", "kernel_ms": hot_avg}
    tr = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tr):
        try:
            t = json.load(open(tr)).get(f"{cfg.name}:{info['variant']}:{n}")
            if t is not None and res["roofline"] is not None:
                res["roofline"]["traffic"] = t
        except Exception:
            pass
    if proba and classif:
        pout = torch.empty((n, cfg.n_classes if cfg.n_classes > 1 else 2), device=dev)
        pm, _, _, _ = time_steps(lambda: model.predict_proba(X, out=pout), steps, args.warmup, dev, world, flush, st)
        res["predict_proba"] = {"value": n_total / (pm / 1e3), "unit": "rows/s", "ms_per_step": pm}

    # ---- e2e through the public host-buffer API
    if args.e2e_steps > 0:
        import torch.distributed as dist
        Xh = torch.empty((n, cfg.n_features), dtype=torch.float32).pin_memory()
        Xh.copy_(X)              # the same seeded rows (the generator is bit-identical on host and device)
        del X
        torch.cuda.empty_cache()
        if tsp is not None:
            e2e_call = lambda: tsp.predict_host(Xh)
            r0, r1 = tsp.slice_of(n)
            d2h = (r1 - r0) * (4 if classif else 4 * cfg.n_classes)
        else:
            oh = (torch.empty(n, dtype=torch.int32) if classif else torch.empty((n, cfg.n_classes))).pin_memory()
            e2e_call = lambda: model.predict_host(Xh, out=oh)
            d2h = int(oh.numel() * oh.element_size())
        e2e_call()
        times = []
        for _ in range(args.e2e_steps):
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            e2e_call()
            times.append(time.perf_counter() - t0)
        # median over the e2e steps: host-side timing on a shared box is noisy
        te = torch.tensor([statistics.median(times)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        res["e2e"] = {"value": n_total / te.item(), "unit": "rows/s",
                      "h2d_bytes_per_step": n * cfg.n_features * 4, "d2h_bytes_per_step": d2h,
                      "api": ("TreeShardedPredictor.predict_host (pinned H2D of all rows per rank -> partials -> "
                              "NCCL reduce-scatter -> finalize -> D2H of the own slice)" if tsp is not None else
                              "bridger_predict_host (2-stream chunked H2D / compute / D2H pipeline)"),
                      "per_rank": "h2d/d2h bytes are per rank"}
    return res, cfg, m, model


def dry_run(args):
    """--dry-run (CPU tests): the launcher and sharding bookkeeping without a
    GPU -- gloo process group, each rank's row shard / tree range, the
    max-over-ranks reduction of a stand-in time; rank 0 prints one JSON line."""
    import torch
    import torch.distributed as dist
    from synth import CONFIGS
    world, rank, _ = dist_env()
    if world > 1:
        dist.init_process_group("gloo")
    cfg = CONFIGS[args.config]
    if cfg.sharding == "trees":
        part = (0, cfg.n_rows)
    else:
        part = row_range(cfg.n_rows, world, rank)
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    shards = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_gather(shards, torch.tensor(part, dtype=torch.int64))
    else:
        shards = [torch.tensor(part, dtype=torch.int64)]
    if rank == 0:
        print(json.dumps({"dry_run": True, "metric": METRIC, "n_gpus": world, "config": workload_config(cfg, world),
                          "row_shards": [s.tolist() for s in shards], "max_over_ranks": t.item()}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main(argv=None):
    argv = list(sys.argv[1:] if argv is None else argv)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C3")
    ap.add_argument("--variant", default=None, choices=[None, "auto", "traverse", "gemm", "gemm_staged"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-gemm", action="store_true", help="skip the GEMM-form (tcgen05) sub-measurement")
    ap.add_argument("--no-extra", action="store_true", help="skip the C2 / C4-1M / C5-shard sub-measurements")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--rows", type=int, default=None, help="override total rows (exploration; reported in config)")
    ap.add_argument("--trees", type=int, default=None, help="override ensemble size (exploration)")
    ap.add_argument("--dry-run", action="store_true", help="CPU: launcher + sharding bookkeeping only (tests)")
    ap.add_argument("--no-fused-reduce", action="store_true",
                    help="tree sharding: NCCL reduce-scatter instead of the fused peer-memory reduce")
    args = ap.parse_args(argv)
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference(args)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return relaunch(argv, args.gpus)
    if args.dry_run:
        return dry_run(args)

    import torch
    import torch.distributed as dist

    import paper_2405_12491_b200 as B

    world, rank, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if torch.cuda.device_count() < world and world > 1:
        raise SystemExit(f"{world} ranks need {world} GPUs; this box has {torch.cuda.device_count()}")
    torch.cuda.set_device(local)
    if world > 1:
        # bind the process group to this rank's GPU before the first collective
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)

    res, cfg, m, model = run_workload(args.config, args, dev, world, rank, local, headline=True,
                                         rows=args.rows, trees=args.trees, proba=False)
    line = {
        "metric": METRIC, "value": res["value"], "unit": "rows/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": res["ms_per_step"], "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": res["dtype"],
        "data": "synthetic (counter-based seeded generator; random calibrated trees of the config's shape)",
        "config": res["config"], "variant": res["variant"], "exact_tier": res["exact_tier"],
        "gpu_launches": res["gpu_launches"], "wall_s_timed": res["wall_s_timed"], "roofline": res["roofline"],
        "e2e": res.get("e2e"), "clocks": res.get("clocks"), "setup_s": res.get("setup_s"),
    }
    model.close()
    if world == 1 and rank == 0 and not args.no_gemm and cfg.depth <= 8:
        from synth import gen_x_torch
        Xg = gen_x_torch(cfg.seed, 0, min(cfg.n_rows, 2_000_000), cfg.n_features, device=dev)
        line["path_contraction"] = gemm_roofline(B, m, cfg, Xg, dev)
        del Xg
    if world == 1 and not args.no_extra and args.rows is None and args.trees is None and args.config == "C3":
        extra = {}
        torch.cuda.empty_cache()
        for key, name, rows, trees, pr in (("C1_latency", "C1", None, None, False), ("C2", "C2", None, None, True),
                                           ("C4_1M_rows", "C4", 1_000_000, None, True),
                                           ("C5_shard_1250_trees_1M_rows", "C5", 1_000_000, 1250, False)):
            sub = argparse.Namespace(**vars(args))
            sub.e2e_steps = 0
            r, _, _, mm = run_workload(name, sub, dev, 1, 0, local, headline=False, rows=rows, trees=trees,
                                          proba=pr)
            mm.close()
            torch.cuda.empty_cache()
            r.pop("wall_s_timed", None)
            if name == "C1":  # one 150-row decision tree: a latency figure
                r["latency_us"] = r["ms_per_step"] * 1e3
            extra[key] = r
        line["extra"] = extra
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(m, cfg)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())

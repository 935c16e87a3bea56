"""Multi-GPU orchestration of the tree-ensemble hot path.

One process per GPU (torchrun), ``torch.distributed`` for the plumbing.

* Row sharding (C2..C4): contiguous row shards, the full model resident on
  every GPU, NO data-path collective -- rows are independent units, so the
  concatenation of the shards' outputs equals the single-GPU output bitwise.
* Tree sharding (C5, ensembles too large or too slow for one GPU): rank r holds
  a contiguous, visit-balanced slice of the trees, computes raw per-row partial
  sums for ALL rows (``bridger_predict_raw``: int64 fixed point at the WHOLE
  ensemble's exponent q, reading c9), then ONE ``reduce_scatter`` SUM over
  NVLink/NVSwitch leaves each rank the exact totals of its row slice, which it
  finalises locally (``bridger_finalize``).  int64 addition is associative, so
  the result is independent of NCCL's ring/tree/NVLS choice and bitwise equal
  to the single-GPU run in tiers E53/E63.

The partition helpers are pure Python and tested on CPU; the collective goes
through ``torch.distributed`` (NCCL on GPUs; the gloo path used by the CPU
tests emulates reduce-scatter with all_reduce + slice because gloo lacks it).
"""
from __future__ import annotations

from typing import List, Sequence, Tuple

import numpy as np

TIER_CODE = {"E53": 0, "E63": 1, "F64": 2}


def row_range(n_rows: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous row shard [a, b) of rank (balanced, ceil-first)."""
    per = -(-n_rows // world)
    a = min(n_rows, rank * per)
    return a, min(n_rows, a + per)


def tree_visits(desc) -> np.ndarray:
    """Per-tree traversal cost: the longest root-to-leaf path (node visits per
    row), at least 1.  Vectorised (pointer jumping over parent links), so a
    10,000-tree depth-10 ensemble costs milliseconds, not a Python walk."""
    offs = np.asarray(desc.tree_offsets, np.int64)
    left = np.asarray(desc.left, np.int64)
    right = np.asarray(desc.right, np.int64)
    n = int(offs[-1])
    T = len(offs) - 1
    if T == 0:
        return np.zeros(0, np.int64)
    base = np.repeat(offs[:-1], np.diff(offs))          # tree offset of every node
    parent = np.full(n, -1, np.int64)
    inner = np.nonzero(left >= 0)[0]
    parent[left[inner] + base[inner]] = inner
    parent[right[inner] + base[inner]] = inner
    # invariant: depth[v] = edges from v to jump[v] (jump[v] >= 0), else v's depth
    depth = (parent >= 0).astype(np.int64)
    jump = parent.copy()
    while True:
        live = np.nonzero(jump >= 0)[0]
        if live.size == 0:
            break
        up = jump[live]
        d_up, j_up = depth[up].copy(), jump[up].copy()   # simultaneous update
        depth[live] += d_up
        jump[live] = j_up
    best = np.maximum.reduceat(depth, offs[:-1]) if n else np.zeros(T, np.int64)
    return np.maximum(best, 1)


def tree_partition(costs: Sequence[int], world: int) -> List[Tuple[int, int]]:
    """Split trees [0, T) into `world` contiguous ranges of near-equal total
    cost.  When T >= world every range holds at least one tree (bounds are
    clamped to [previous + 1, T - (ranks left)]), so no rank is left without
    work whatever the cost skew; T < world raises on every rank alike."""
    costs = np.asarray(costs, np.int64)
    T = len(costs)
    if T < world:
        raise ValueError(f"{world} ranks but only {T} trees: every tree shard needs >= 1 tree")
    cum = np.concatenate([[0], np.cumsum(costs)])
    total = cum[-1]
    bounds = [0]
    for r in range(1, world):
        target = total * r / world
        j = int(np.searchsorted(cum, target, side="left"))
        j = max(bounds[-1] + 1, min(T - (world - r), j))
        bounds.append(j)
    bounds.append(T)
    return [(bounds[r], bounds[r + 1]) for r in range(world)]


def _reduce_scatter_sum(out, inp, group=None):
    import torch.distributed as dist
    if dist.get_backend(group) == "nccl":
        dist.reduce_scatter_tensor(out, inp, op=dist.ReduceOp.SUM, group=group)
    else:
        # gloo (CPU tests, and multi-rank tests sharing one GPU): host-side
        # all_reduce + own slice.  The partials are staged through host memory
        # so no collective ever runs on (or waits inside) the device.
        buf = inp.detach().to("cpu", copy=True)
        dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
        r = dist.get_rank(group)
        out.copy_(buf.view(dist.get_world_size(group), -1)[r].view(out.shape))
    return out


def reduce_scatter_rows(raw, group=None):
    """raw [N_pad, K] partial sums on every rank -> this rank's row slice of the
    SUM over ranks.  N_pad must be a multiple of the world size."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    n = raw.shape[0]
    assert n % world == 0, "pad rows to a multiple of the world size"
    out = torch.empty((n // world,) + tuple(raw.shape[1:]), dtype=raw.dtype, device=raw.device)
    return _reduce_scatter_sum(out, raw.contiguous(), group)


def _pinned_host(x):
    import torch
    if isinstance(x, np.ndarray):
        x = torch.from_numpy(np.ascontiguousarray(x, np.float32))
    return x if x.is_pinned() else x.pin_memory()


class RowShardedPredictor:
    """Full model on every rank; each rank predicts its own contiguous rows
    [row_range(N, world, rank)) -- no data-path collective."""

    def __init__(self, desc, device: int, variant=None, group=None):
        import torch.distributed as dist

        from . import Model
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.model = Model(desc, device=device, variant=variant)

    def rows(self, n_rows: int) -> Tuple[int, int]:
        return row_range(n_rows, self.world, self.rank)

    def predict(self, X_local, proba: bool = False):
        return self.model.predict_proba(X_local) if proba else self.model.predict(X_local)

    def predict_host(self, X_host_local, proba: bool = False, out=None):
        """End to end on this rank's host rows (pinned H2D, predict, D2H)."""
        return self.model.predict_host(X_host_local, proba=proba, out=out)


class TreeShardedPredictor:
    """Rank r holds trees [a_r, b_r); raw partials are reduce-scattered by row."""

    def __init__(self, desc, device: int, group=None, variant=None):
        import torch.distributed as dist

        from . import Model, analyze_exactness
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.device = int(device)
        q, tier, _ = analyze_exactness(desc)          # of the WHOLE ensemble
        self.total_trees = len(desc.tree_offsets) - 1
        self.ranges = tree_partition(tree_visits(desc), self.world)   # raises alike on every rank
        a, b = self.ranges[self.rank]
        self.model = Model(_subset(desc, range(a, b)), device=device, force_fixed_point=(q, TIER_CODE[tier]),
                           variant=variant)
        self._xbuf = None

    def slice_of(self, n_rows: int) -> Tuple[int, int]:
        """Rows [row0, row1) this rank owns after the reduce-scatter."""
        n_pad = -(-n_rows // self.world) * self.world
        row0 = self.rank * (n_pad // self.world)
        return min(row0, n_rows), min(n_rows, row0 + n_pad // self.world)

    def _reduce_finalize(self, raw, n, proba):
        import torch
        n_pad = -(-n // self.world) * self.world
        if n_pad != n:
            raw = torch.cat([raw, torch.zeros((n_pad - n, raw.shape[1]), dtype=raw.dtype, device=raw.device)])
        mine = reduce_scatter_rows(raw, self.group)
        row0, row1 = self.slice_of(n)
        return row0, self.model.finalize(mine[: row1 - row0].contiguous(), total_trees=self.total_trees, proba=proba)

    def predict(self, X_all, proba: bool = False):
        """X_all: the same [N, F] rows on every rank.  Returns (row0, outputs of
        this rank's row slice [row0, row0 + N_pad/world) clipped to N)."""
        return self._reduce_finalize(self.model.predict_raw(X_all), X_all.shape[0], proba)

    def predict_host(self, X_host, proba: bool = False):
        """End to end from HOST rows: pinned H2D of X on every rank, partial
        sums, ONE reduce-scatter, finalize of the own slice, D2H of it.
        Returns (row0, host outputs of this rank's slice)."""
        import torch
        X_host = _pinned_host(X_host)
        dev = torch.device("cuda", self.device)
        if self._xbuf is None or self._xbuf.shape != X_host.shape:
            self._xbuf = torch.empty(X_host.shape, dtype=torch.float32, device=dev)
        self._xbuf.copy_(X_host, non_blocking=True)
        row0, out = self.predict(self._xbuf, proba=proba)
        host = torch.empty(out.shape, dtype=out.dtype).pin_memory()
        host.copy_(out, non_blocking=True)
        torch.cuda.current_stream(dev).synchronize()
        return row0, host


class FusedTreeShardedPredictor(TreeShardedPredictor):
    """Tree sharding with the reduce-scatter fused into the walk: every rank's
    K4d kernel adds each row's int64 partial straight into the accumulator
    slice of the rank that owns the row -- its own memory or a peer's, opened
    through CUDA IPC and written over NVLink P2P (red.global.add.u64,
    bridger_predict_raw_scatter).  No separate collective kernel and no
    partial array: the data movement overlaps the walk tile by tile.  Per
    call: zero own slice -> barrier -> walk+scatter -> barrier -> finalize own
    slice; the host barriers are the only cross-rank synchronisation (no
    kernel ever waits for another rank).  Slices are bitwise equal to the NCCL
    path's (int64 addition is associative).  Needs peer access between the
    ranks' devices (same device is fine) and the multi-chunk coded exact
    layout; ``available`` says whether both hold."""

    def __init__(self, desc, device: int, group=None, variant=None):
        super().__init__(desc, device=device, group=group, variant=variant)
        import torch
        import torch.distributed as dist
        self._slice = None
        self._ptrs = None
        self._peers = []
        lay = self.model.layout()
        ok = lay["format"] == "codes_deep" and self.model.info()["acc_is_int64"]
        devs = [None] * self.world
        dist.all_gather_object(devs, self.device, group=group)
        for d in devs:
            if d != self.device and not torch.cuda.can_device_access_peer(self.device, d):
                ok = False
        flags = [None] * self.world
        dist.all_gather_object(flags, bool(ok), group=group)
        self.available = all(flags)

    def _ensure(self, rpr: int):
        """Own slice of >= rpr rows; exchange IPC handles when it (re)grows."""
        import torch
        import torch.distributed as dist
        from torch.multiprocessing.reductions import reduce_tensor
        if self._slice is not None and self._slice.shape[0] >= rpr:
            return
        K = self.model.n_outputs
        self._slice = torch.zeros((rpr, K), dtype=torch.int64, device=torch.device("cuda", self.device))
        handles = [None] * self.world
        dist.all_gather_object(handles, reduce_tensor(self._slice), group=self.group)
        self._peers = []
        ptrs = []
        for r, (fn, args) in enumerate(handles):
            if r == self.rank:
                ptrs.append(self._slice.data_ptr())
            else:
                t = fn(*args)   # peer slice mapped into this process (CUDA IPC)
                self._peers.append(t)
                ptrs.append(t.data_ptr())
        self._ptrs = ptrs

    def predict(self, X_all, proba: bool = False):
        import torch
        import torch.distributed as dist
        if not self.available:
            return super().predict(X_all, proba=proba)
        n = X_all.shape[0]
        rpr = -(-n // self.world)
        rpr = -(-rpr // 32) * 32
        self._ensure(rpr)
        dev = torch.device("cuda", self.device)
        self._slice.zero_()
        torch.cuda.current_stream(dev).synchronize()
        dist.barrier(group=self.group)            # every slice zeroed before any rank adds
        self.model.predict_raw_scatter(X_all, self._ptrs, rpr)
        torch.cuda.current_stream(dev).synchronize()
        dist.barrier(group=self.group)            # every rank's adds landed
        row0 = min(self.rank * rpr, n)
        row1 = min(n, row0 + rpr)
        out = self.model.finalize(self._slice[: row1 - row0], total_trees=self.total_trees, proba=proba)
        return row0, out

    def slice_of(self, n_rows: int) -> Tuple[int, int]:
        if not self.available:
            return super().slice_of(n_rows)
        rpr = -(-(-(-n_rows // self.world)) // 32) * 32
        row0 = min(self.rank * rpr, n_rows)
        return row0, min(n_rows, row0 + rpr)


def _subset(desc, trees):
    """Model made of the listed trees (node arrays re-based); desc-agnostic.
    Honours per-tree scalar outputs (``tree_output``, reading c15): such models
    store ONE value per node, otherwise K."""
    from types import SimpleNamespace
    trees = list(trees)
    if not trees:
        raise ValueError("empty tree subset")
    offs = np.asarray(desc.tree_offsets, np.int64)
    K = int(desc.n_outputs)
    tout = getattr(desc, "tree_output", None)
    vw = 1 if tout is not None else K
    idx = np.concatenate([np.arange(offs[t], offs[t + 1]) for t in trees])
    sizes = [int(offs[t + 1] - offs[t]) for t in trees]
    new_offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    val = np.asarray(desc.value, np.float32).reshape(-1, vw)[idx].reshape(-1)
    ml = getattr(desc, "missing_left", None)
    return SimpleNamespace(
        n_features=desc.n_features, n_outputs=K, tree_offsets=new_offs,
        feature=np.asarray(desc.feature)[idx], threshold=np.asarray(desc.threshold)[idx],
        left=np.asarray(desc.left)[idx], right=np.asarray(desc.right)[idx], value=val,
        missing_left=None if ml is None else np.asarray(ml)[idx], task=getattr(desc, "task", 0),
        agg=getattr(desc, "agg", 0), post=getattr(desc, "post", 0), base_score=getattr(desc, "base_score", None),
        leaf_scale=getattr(desc, "leaf_scale", 1.0),
        tree_output=None if tout is None else np.asarray(tout, np.int32)[trees])


# ------------------------------------------------------------- 2-D sharding --
def grid_2d(world: int, row_groups: int, rank: int):
    """Rank -> (row group rg, tree group tg) for a rows x trees process grid:
    rank = rg * TG + tg with TG = world // row_groups."""
    if world % row_groups:
        raise ValueError("world size must be a multiple of row_groups")
    tg_n = world // row_groups
    return rank // tg_n, rank % tg_n, tg_n


def make_row_group_comms(world: int, row_groups: int):
    """One communicator per row group (its TG tree-shard ranks).  Every rank
    must call this with the same arguments (torch.distributed.new_group is
    collective); returns the list of groups, index rg."""
    import torch.distributed as dist
    tg_n = world // row_groups
    return [dist.new_group(list(range(rg * tg_n, (rg + 1) * tg_n))) for rg in range(row_groups)]


class TwoDShardedPredictor:
    """rows x trees sharding (§8(f4)) for ensembles both huge and wide: the
    row group rg owns rows shard rg, the tree group tg trees shard tg; raw int64
    partials are reduce-scattered inside the row group only (TG ranks)."""

    def __init__(self, desc, device: int, row_groups: int):
        import torch.distributed as dist

        from . import Model, analyze_exactness
        world, rank = dist.get_world_size(), dist.get_rank()
        self.rg, self.tg, self.tg_n = grid_2d(world, row_groups, rank)
        self.comms = make_row_group_comms(world, row_groups)
        q, tier, _ = analyze_exactness(desc)
        self.total_trees = len(desc.tree_offsets) - 1
        a, b = tree_partition(tree_visits(desc), self.tg_n)[self.tg]   # raises alike on every rank
        self.model = Model(_subset(desc, range(a, b)), device=device, force_fixed_point=(q, TIER_CODE[tier]))

    def predict(self, X_rows, proba: bool = False):
        """X_rows: the row group's rows (same on its TG ranks).  Returns (row0
        within the row group's rows, outputs of this rank's slice)."""
        import torch
        n = X_rows.shape[0]
        n_pad = -(-n // self.tg_n) * self.tg_n
        raw = self.model.predict_raw(X_rows)
        if n_pad != n:
            raw = torch.cat([raw, torch.zeros((n_pad - n, raw.shape[1]), dtype=raw.dtype, device=raw.device)])
        mine = reduce_scatter_rows(raw, self.comms[self.rg])
        row0 = self.tg * (n_pad // self.tg_n)
        keep = max(0, min(mine.shape[0], n - row0))
        return row0, self.model.finalize(mine[:keep].contiguous(), total_trees=self.total_trees, proba=proba)

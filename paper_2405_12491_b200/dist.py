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
    """Per-tree traversal cost (padded depth = node visits per row)."""
    offs = np.asarray(desc.tree_offsets)
    left = np.asarray(desc.left)
    out = np.zeros(len(offs) - 1, np.int64)
    for t in range(len(offs) - 1):
        a, b = int(offs[t]), int(offs[t + 1])
        l, r = left[a:b], np.asarray(desc.right)[a:b]
        depth = np.zeros(b - a, np.int64)
        stack = [0]
        best = 0
        while stack:
            n = stack.pop()
            if l[n] == -1:
                best = max(best, depth[n])
            else:
                depth[l[n]] = depth[r[n]] = depth[n] + 1
                stack += [int(l[n]), int(r[n])]
        out[t] = max(best, 1)
    return out


def tree_partition(costs: Sequence[int], world: int) -> List[Tuple[int, int]]:
    """Split trees [0, T) into `world` contiguous ranges of near-equal total cost."""
    costs = np.asarray(costs, np.int64)
    T = len(costs)
    cum = np.concatenate([[0], np.cumsum(costs)])
    total = cum[-1]
    bounds = [0]
    for r in range(1, world):
        target = total * r / world
        j = int(np.searchsorted(cum, target, side="left"))
        j = max(bounds[-1], min(T, j))
        bounds.append(j)
    bounds.append(T)
    return [(bounds[r], bounds[r + 1]) for r in range(world)]


def _reduce_scatter_sum(out, inp, group=None):
    import torch.distributed as dist
    if dist.get_backend(group) == "nccl":
        dist.reduce_scatter_tensor(out, inp, op=dist.ReduceOp.SUM, group=group)
    else:  # gloo (CPU tests): all_reduce + own slice
        buf = inp.clone()
        dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
        r = dist.get_rank(group)
        out.copy_(buf.view(dist.get_world_size(group), -1)[r].view_as(out))
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


class RowShardedPredictor:
    """Full model on every rank; each rank predicts its own contiguous rows."""

    def __init__(self, desc, device: int, variant=None):
        from . import Model
        self.model = Model(desc, device=device, variant=variant)

    def predict(self, X_local, proba: bool = False):
        return self.model.predict_proba(X_local) if proba else self.model.predict(X_local)


class TreeShardedPredictor:
    """Rank r holds trees [a_r, b_r); raw partials are reduce-scattered by row."""

    def __init__(self, desc, device: int, group=None):
        import torch.distributed as dist

        from . import Model, analyze_exactness
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        q, tier, _ = analyze_exactness(desc)          # of the WHOLE ensemble
        self.total_trees = len(desc.tree_offsets) - 1
        self.ranges = tree_partition(tree_visits(desc), self.world)
        a, b = self.ranges[self.rank]
        if b <= a:
            raise ValueError("more ranks than trees")
        self.model = Model(_subset(desc, range(a, b)), device=device, force_fixed_point=(q, TIER_CODE[tier]))

    def predict(self, X_all, proba: bool = False):
        """X_all: the same [N, F] rows on every rank.  Returns (row0, outputs of
        this rank's row slice [row0, row0 + N_pad/world) clipped to N)."""
        import torch
        n = X_all.shape[0]
        n_pad = -(-n // self.world) * self.world
        raw = self.model.predict_raw(X_all)
        if n_pad != n:
            raw = torch.cat([raw, torch.zeros((n_pad - n, raw.shape[1]), dtype=raw.dtype, device=raw.device)])
        mine = reduce_scatter_rows(raw, self.group)
        row0 = self.rank * (n_pad // self.world)
        keep = max(0, min(mine.shape[0], n - row0))
        out = self.model.finalize(mine[:keep].contiguous(), total_trees=self.total_trees, proba=proba)
        return row0, out


def _subset(desc, trees):
    """Model made of the listed trees (node arrays re-based); desc-agnostic."""
    from types import SimpleNamespace
    trees = list(trees)
    offs = np.asarray(desc.tree_offsets, np.int64)
    K = int(desc.n_outputs)
    idx = np.concatenate([np.arange(offs[t], offs[t + 1]) for t in trees])
    sizes = [int(offs[t + 1] - offs[t]) for t in trees]
    new_offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    val = np.asarray(desc.value, np.float32).reshape(-1, K)[idx].reshape(-1)
    ml = getattr(desc, "missing_left", None)
    return SimpleNamespace(
        n_features=desc.n_features, n_outputs=K, tree_offsets=new_offs,
        feature=np.asarray(desc.feature)[idx], threshold=np.asarray(desc.threshold)[idx],
        left=np.asarray(desc.left)[idx], right=np.asarray(desc.right)[idx], value=val,
        missing_left=None if ml is None else np.asarray(ml)[idx], task=getattr(desc, "task", 0),
        agg=getattr(desc, "agg", 0), post=getattr(desc, "post", 0), base_score=getattr(desc, "base_score", None),
        leaf_scale=getattr(desc, "leaf_scale", 1.0))


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
        a, b = tree_partition(tree_visits(desc), self.tg_n)[self.tg]
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

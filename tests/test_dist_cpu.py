"""Multi-GPU bookkeeping on CPU with gloo, world_size 2:
row shards need no collective and concatenate to the full result; tree shards'
int64 fixed-point partials (at the WHOLE ensemble's q, reading c9) reduce-
scattered by row equal the full-ensemble sums exactly; partitions are
contiguous, complete and balanced."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import paper_2405_12491_b200 as B
from paper_2405_12491_b200.dist import (grid_2d, make_row_group_comms, reduce_scatter_rows, row_range,
                                        tree_partition, tree_visits)
from paper_2405_12491_b200.dist import _subset
from synth import gen_x, make_config, multiclass_gbdt, perfect_ensemble, prune_ensemble


def test_row_range_covers_exactly():
    for n in (0, 1, 7, 1000, 1001):
        for w in (1, 2, 3, 8):
            parts = [row_range(n, w, r) for r in range(w)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            for (a, b), (c, d) in zip(parts, parts[1:]):
                assert b == c and a <= b


def test_tree_partition_balanced_contiguous():
    m = prune_ensemble(perfect_ensemble(3, 57, 7, 5, calib_rows=256), 3, p=0.3)
    cost = tree_visits(m)
    for w in (1, 2, 4, 8):
        parts = tree_partition(cost, w)
        assert parts[0][0] == 0 and parts[-1][1] == m.n_trees
        assert all(b == c for (_, b), (c, _) in zip(parts, parts[1:]))
        loads = [cost[a:b].sum() for a, b in parts]
        assert max(loads) - min(loads) <= 2 * cost.max()


def test_tree_partition_nonempty_under_skew():
    # costs [8, 8, 1, 1] on 4 ranks used to give an empty range
    for costs, w in (([8, 8, 1, 1], 4), ([100, 1, 1, 1, 1], 5), ([1] * 7 + [50], 8), ([3, 3], 2)):
        parts = tree_partition(costs, w)
        assert all(b > a for a, b in parts), parts
        assert parts[0][0] == 0 and parts[-1][1] == len(costs)
        assert all(b == c for (_, b), (c, _) in zip(parts, parts[1:]))
    with pytest.raises(ValueError):
        tree_partition([1, 2, 3], 4)


def test_subset_keeps_scalar_tree_outputs():
    """Round-1 bug: ``_subset`` reshaped scalar leaves as K-vectors and dropped
    tree_output (multiclass boosting, reading c15).  The shard must equal the
    same trees taken by ModelDesc.subset, and the shards' oracle sums add up
    to the whole ensemble's."""
    m = multiclass_gbdt(81, 30, 6, 14, 5)
    X = gen_x(82, 0, 97, 14)
    full = oracle.run(m, X)["acc"]
    tot = np.zeros_like(full)
    for a, b in tree_partition(tree_visits(m), 3):
        sub = _subset(m, range(a, b))
        ref = m.subset(range(a, b))
        assert len(sub.value) == len(ref.value) == int(ref.tree_offsets[-1])
        np.testing.assert_array_equal(sub.tree_output, np.arange(a, b) % 5)
        acc = oracle.run(sub, X)["acc"]
        np.testing.assert_array_equal(acc, oracle.run(ref, X)["acc"])
        tot += acc
    np.testing.assert_allclose(tot, full, rtol=1e-12, atol=1e-12)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # tree sharding
        m = perfect_ensemble(5, 23, 6, 9, kind="regression", lr=0.05, calib_rows=512)
        m = prune_ensemble(m, 5, p=0.2)
        X = gen_x(6, 0, 301, 9)          # 301 rows: padded to a multiple of world
        qx, tier, _ = B.analyze_exactness(m)
        a, b = tree_partition(tree_visits(m), world)[rank]
        part = oracle.run(m.subset(range(a, b)), X)["acc"]
        raw = torch.from_numpy(np.round(np.ldexp(part, -qx)).astype(np.int64))
        n_pad = -(-X.shape[0] // world) * world
        raw = torch.cat([raw, torch.zeros((n_pad - X.shape[0], 1), dtype=torch.int64)])
        mine = reduce_scatter_rows(raw)
        full = oracle.run(m, X)["acc"]
        want = np.round(np.ldexp(full, -qx)).astype(np.int64)
        r0 = rank * (n_pad // world)
        keep = min(mine.shape[0], X.shape[0] - r0)
        np.testing.assert_array_equal(mine[:keep].numpy(), want[r0:r0 + keep])
        # row sharding: no collective on the data path; gather only to check
        _, mc = make_config("C2", n_trees=7)
        Xc = gen_x(2, 0, 257, 28)
        ra, rb = row_range(Xc.shape[0], world, rank)
        lab = torch.from_numpy(oracle.run(mc, Xc[ra:rb])["label"].astype(np.int64))
        sizes = [row_range(Xc.shape[0], world, r) for r in range(world)]
        mx = max(b_ - a_ for a_, b_ in sizes)
        padded = torch.cat([lab, torch.full((mx - lab.shape[0],), -1, dtype=torch.int64)])
        bufs = [torch.zeros(mx, dtype=torch.int64) for _ in sizes]
        dist.all_gather(bufs, padded)
        got = torch.cat([bb[: b_ - a_] for bb, (a_, b_) in zip(bufs, sizes)])
        np.testing.assert_array_equal(got.numpy(), oracle.run(mc, Xc)["label"])
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_tree_and_row_sharding():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res


def _worker_2d(rank, world, port, q):
    """rows x trees grid 2 x 2: each row group reduce-scatters its tree shards'
    exact int64 partials among its own 2 ranks."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        row_groups = 2
        rg, tg, tg_n = grid_2d(world, row_groups, rank)
        comms = make_row_group_comms(world, row_groups)
        m = perfect_ensemble(7, 19, 5, 6, kind="regression", lr=0.05, calib_rows=512)
        m = prune_ensemble(m, 7, p=0.2)
        X = gen_x(8, 0, 203, 6)
        qx, _, _ = B.analyze_exactness(m)
        ra, rb = row_range(X.shape[0], row_groups, rg)
        Xg = X[ra:rb]
        a, b = tree_partition(tree_visits(m), tg_n)[tg]
        part = oracle.run(m.subset(range(a, b)), Xg)["acc"]
        raw = torch.from_numpy(np.round(np.ldexp(part, -qx)).astype(np.int64))
        n = Xg.shape[0]
        n_pad = -(-n // tg_n) * tg_n
        raw = torch.cat([raw, torch.zeros((n_pad - n, 1), dtype=torch.int64)])
        mine = reduce_scatter_rows(raw, comms[rg])
        full = np.round(np.ldexp(oracle.run(m, Xg)["acc"], -qx)).astype(np.int64)
        r0 = tg * (n_pad // tg_n)
        keep = min(mine.shape[0], n - r0)
        np.testing.assert_array_equal(mine[:keep].numpy(), full[r0:r0 + keep])
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_gloo_world4_rows_x_trees_grid():
    assert grid_2d(4, 2, 3) == (1, 1, 2) and grid_2d(8, 2, 5) == (1, 1, 4)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_2d, args=(r, 4, port, q)) for r in range(4)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {r: "ok" for r in range(4)}, res

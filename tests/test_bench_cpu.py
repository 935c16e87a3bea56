"""bench.py's launcher and sharding bookkeeping on CPU:
`--gpus N` outside torchrun starts N ranks itself (torch.distributed.run,
127.0.0.1 rendezvous) and the line reports n_gpus = N; row-sharded configs
split the config's TOTAL rows into contiguous shards (C4: 100M rows, 50M per
rank at 2); tree-sharded C5 gives every rank all rows."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_bench_gpus2_starts_two_ranks_and_splits_total_rows():
    d = _run("--gpus", "2", "--dry-run", "--config", "C4")
    assert d["n_gpus"] == 2
    assert d["row_shards"] == [[0, 50_000_000], [50_000_000, 100_000_000]]
    assert d["max_over_ranks"] == 2.0
    assert d["config"]["n_rows_per_gpu"] == 50_000_000


def test_bench_tree_sharded_every_rank_all_rows():
    d = _run("--gpus", "2", "--dry-run", "--config", "C5")
    assert d["n_gpus"] == 2
    assert d["row_shards"] == [[0, 10_000_000], [0, 10_000_000]]


def test_bench_default_is_c3_single_rank():
    d = _run("--dry-run")
    assert d["n_gpus"] == 1 and d["config"]["workload"].startswith("C3:")
    assert d["row_shards"] == [[0, 10_000_000]]

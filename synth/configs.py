"""BASELINE.json ``configs`` as seeded synthetic workloads.

C1  DT  T=1     D=3   150x4   (iris-shaped, host-generated), K=3 classification
C2  RF  T=100   D=8   1Mx28   binary classification (K=2)       <- bench N=1 workload
C3  GBDT T=500  D=6   10Mx90  regression, lr 0.1, base 0.5
C4  RF  T=1000  D=12  100Mx64 K=8, row-sharded x8
C5  GBDT T=10000 D=10 10Mx200 regression, lr 0.01, tree-sharded x8 + NCCL reduce
"""
from __future__ import annotations

from dataclasses import dataclass

from .trees import perfect_ensemble
from .xgen import iris_like_x


@dataclass(frozen=True)
class Config:
    name: str
    kind: str
    n_trees: int
    depth: int
    n_rows: int
    n_features: int
    n_classes: int
    seed: int
    lr: float = 0.1
    sharding: str = "rows"
    describe: str = ""


CONFIGS = {
    "C1": Config("C1", "classification", 1, 3, 150, 4, 3, 1,
                 describe="single decision tree depth 3 on iris-shaped data (150 rows x 4 features, 3 classes)"),
    "C2": Config("C2", "classification", 100, 8, 1_000_000, 28, 2, 2,
                 describe="random forest 100 trees depth 8, 1M rows x 28 features binary classification"),
    "C3": Config("C3", "regression", 500, 6, 10_000_000, 90, 1, 3, lr=0.1,
                 describe="gradient-boosted trees 500 trees depth 6 regression, 10M rows x 90 features"),
    "C4": Config("C4", "classification", 1000, 12, 100_000_000, 64, 8, 4,
                 describe="random forest 1000 trees depth 12 multiclass (8 classes), 100M rows x 64 features, row-sharded over 8 GPUs"),
    "C5": Config("C5", "regression", 10000, 10, 10_000_000, 200, 1, 5, lr=0.01, sharding="trees",
                 describe="GBDT 10000 trees depth 10 tree-sharded across 8 GPUs with NCCL score reduce, 10M rows x 200 features"),
}


def make_config(name: str, n_trees: int | None = None):
    """(Config, ModelDesc) for a named config; ``n_trees`` shrinks the ensemble
    (parity tests at reduced sizes keep depth, width and value recipe)."""
    c = CONFIGS[name]
    T = c.n_trees if n_trees is None else n_trees
    if name == "C1":
        x = iris_like_x(c.seed, c.n_rows)
        m = perfect_ensemble(c.seed, T, c.depth, c.n_features, kind=c.kind,
                             n_classes=c.n_classes, calib_x=x)
    else:
        m = perfect_ensemble(c.seed, T, c.depth, c.n_features, kind=c.kind,
                             n_classes=c.n_classes, lr=c.lr)
    m.meta["config"] = name
    return c, m

"""Seeded synthetic inputs shared by the oracle-side tests and the CUDA path.

This module is deliberately free of the method's arithmetic: it never walks a
tree to *predict* anything.  It produces

* feature matrices ``X`` from a counter-based generator (SplitMix64 keyed by
  ``(seed, row, col)``), bit-identical on numpy (host) and torch (any device),
  so any row range can be regenerated anywhere (SURVEY.md §8(d) "Concrete
  synthetic inputs");
* tree ensembles in the node-array form of the C ABI (``ModelDesc``), with
  thresholds calibrated on a sample the way a trainer would place them
  (construction, not inference);
* the five BASELINE.json configurations C1..C5 (``configs.py``).

Both ``oracle/`` and ``paper_2405_12491_b200`` receive the same arrays; neither
imports the other.
"""
from .xgen import gen_x, gen_x_torch, splitmix64_np, inject_specials, iris_like_x
from .trees import ModelDesc, multiclass_gbdt, perfect_ensemble, prune_ensemble, stump_model
from .configs import CONFIGS, make_config

__all__ = [
    "gen_x", "gen_x_torch", "splitmix64_np", "inject_specials", "iris_like_x",
    "ModelDesc", "perfect_ensemble", "prune_ensemble", "stump_model",
    "CONFIGS", "make_config",
]

"""Test-side helpers: golden-fixture parsing and model builders (no method arithmetic)."""
import json
import os

import numpy as np

from synth.trees import ModelDesc

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def f32(tok) -> np.float32:
    if isinstance(tok, (int, float)):
        return np.float32(tok)
    tok = str(tok)
    if tok == "sub_min":
        return np.float32(1.4e-45)
    if tok.startswith("next_up:"):
        return np.nextafter(np.float32(tok[8:]), np.float32(np.inf))
    if tok.startswith("next_down:"):
        return np.nextafter(np.float32(tok[10:]), np.float32(-np.inf))
    return np.float32(float(tok))


def load_golden(name):
    with open(os.path.join(GOLDEN, name)) as fh:
        return json.load(fh)


def parse_x(rows):
    return np.array([[f32(t) for t in r] for r in rows], dtype=np.float32)


def model_from_json(d) -> ModelDesc:
    K = int(d["n_outputs"])
    return ModelDesc(
        n_features=int(d["n_features"]), n_outputs=K,
        tree_offsets=np.asarray(d["tree_offsets"], np.int64),
        feature=np.asarray(d["feature"], np.int32),
        threshold=np.array([f32(t) for t in d["threshold"]], np.float32),
        left=np.asarray(d["left"], np.int32), right=np.asarray(d["right"], np.int32),
        value=np.asarray(d["value"], np.float32).reshape(-1),
        task=int(d.get("task", 0)), agg=int(d.get("agg", 0)), post=int(d.get("post", 0)),
        missing_left=None if d.get("missing_left") is None else np.asarray(d["missing_left"], np.uint8),
        base_score=None if d.get("base_score") is None else np.asarray(d["base_score"], np.float64),
        leaf_scale=float(d.get("leaf_scale", 1.0)),
        tree_output=None if d.get("tree_output") is None else np.asarray(d["tree_output"], np.int32))


def model_from_trees(trees, n_features, n_outputs, with_missing, **kw) -> ModelDesc:
    offs = [0]
    for t in trees:
        offs.append(offs[-1] + len(t["feature"]))
    cat = lambda k, dt: np.concatenate([np.asarray(t[k], dt).reshape(-1) for t in trees])
    return ModelDesc(
        n_features=n_features, n_outputs=n_outputs, tree_offsets=np.asarray(offs, np.int64),
        feature=cat("feature", np.int32),
        threshold=np.array([f32(x) for t in trees for x in t["threshold"]], np.float32),
        left=cat("left", np.int32), right=cat("right", np.int32), value=cat("value", np.float32),
        missing_left=cat("missing_left", np.uint8) if with_missing else None, **kw)

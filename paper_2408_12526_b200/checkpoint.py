"""Reader for the reference's JSON checkpoints -> engine weights.

Schemas (restated, not imported): ``dense-model-checkpoint-v1`` (nnkernel.py:471-558) and
``ensemble-checkpoint-v1`` (distill.py:586-612). In "binary" mode arrays are base64 little-endian
float64 (bit exact, nnkernel.py:474-477); in "json" mode decimal lists. Non-finite values are
rejected (nnkernel.py:486-487), as are unknown schemas/kinds (nnkernel.py:535-536, :547).
"""
from __future__ import annotations

import base64
import json

import numpy as np

from .weights import DenseGroupWeights, dense_group_from_arrays

MODEL_SCHEMA = "dense-model-checkpoint-v1"
ENSEMBLE_SCHEMA = "ensemble-checkpoint-v1"


def _decode_array(data, shape, mode: str) -> np.ndarray:
    if mode == "binary":
        arr = np.frombuffer(base64.b64decode(data), dtype="<f8").astype(np.float64)
    elif mode == "json":
        arr = np.asarray(data, dtype=np.float64)
    else:
        raise ValueError(f"unknown checkpoint mode {mode!r}")
    arr = arr.reshape(shape)
    if not np.isfinite(arr).all():
        raise ValueError("checkpoint contains non-finite values")
    return arr


def _layer(d: dict, mode: str) -> tuple[np.ndarray, np.ndarray, str]:
    shape = (d["out_dim"], d["in_dim"])
    return (_decode_array(d["weight"], shape, mode), _decode_array(d["bias"], (d["out_dim"],), mode),
            d["activation"])


def _student_layers(d: dict) -> list[tuple[np.ndarray, np.ndarray]]:
    if d.get("schema") != MODEL_SCHEMA:
        raise ValueError(f"not a model checkpoint (schema {d.get('schema')!r})")
    if d["kind"] != "student":
        raise ValueError(f"expected a student checkpoint, got kind {d['kind']!r}")
    mode = d["mode"]
    layers = [_layer(d["input_proj"], mode)] + [_layer(l, mode) for l in d["layers"]]
    for _, _, act in layers:
        if act != "tanh":
            raise ValueError("engine dense students use tanh on every layer (nnkernel.py:272-273)")
    return [(w, b) for w, b, _ in layers]


def ensemble_arrays_from_dict(d: dict):
    """(students, multipliers, classifier) as float64 arrays from an ensemble-checkpoint-v1 dict."""
    if d.get("schema") != ENSEMBLE_SCHEMA:
        raise ValueError("not an ensemble checkpoint")
    students = [_student_layers(s) for s in d["students"]]
    clf = None
    if d["classifier"] is not None:
        w, b, act = _layer(d["classifier"], d["mode"])
        if act != "identity":
            raise ValueError("classifier must be an identity layer (distill.py:535)")
        clf = (w, b)
    return students, list(d["multipliers"]), clf


def load_ensemble_weights(path) -> DenseGroupWeights:
    with open(path, "r", encoding="utf-8") as fh:
        d = json.load(fh)
    return dense_group_from_arrays(*ensemble_arrays_from_dict(d))

"""Float64 restatement of the reference's group forward (dense StudentModel kind).

TEST INFRASTRUCTURE (see oracle/__init__.py). Each function cites the reference lines it follows.
"""
from __future__ import annotations

import numpy as np

TANH = "tanh"
IDENTITY = "identity"


def dense_layer(weight: np.ndarray, bias: np.ndarray, x: np.ndarray, activation: str = TANH) -> np.ndarray:
    """act(x @ W.T + b) — DenseLayer.forward (nnkernel.py:66-76), incl. 1-D squeeze and width check."""
    x = np.asarray(x, dtype=np.float64)
    squeeze = x.ndim == 1
    if squeeze:
        x = x[None, :]
    weight = np.asarray(weight, dtype=np.float64)
    if x.ndim != 2 or x.shape[1] != weight.shape[1]:
        raise ValueError(f"input width {x.shape} does not match layer in_dim {weight.shape[1]}")
    z = x @ weight.T + np.asarray(bias, dtype=np.float64)
    if activation == TANH:
        out = np.tanh(z)
    elif activation == IDENTITY:
        out = z
    else:
        raise ValueError(f"unknown activation {activation!r}")
    return out[0] if squeeze else out


def student_forward(layers: list[tuple[np.ndarray, np.ndarray]], x: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """StudentModel.forward (nnkernel.py:289-301): tanh input_proj, then tanh layers; returns
    (final, mid) with mid tapped after layer ceil(depth/2) (nnkernel.py:280-283)."""
    if len(layers) < 3:
        raise ValueError("student needs at least 2 layers")
    depth = len(layers) - 1
    mid_index = (depth + 1) // 2
    x = np.asarray(x, dtype=np.float64)
    squeeze = x.ndim == 1
    h = dense_layer(*layers[0], x[None, :] if squeeze else x, TANH)
    mid = None
    for i, (w, b) in enumerate(layers[1:], start=1):
        h = dense_layer(w, b, h, TANH)
        if i == mid_index:
            mid = h
    if squeeze:
        return h[0], mid[0]
    return h, mid


def ensemble_rep(finals: list[np.ndarray], multipliers, k: int | None = None) -> np.ndarray:
    """EnsembleState.rep (distill.py:169-178): sum_{m<k} alpha_m * S_m, accumulated left to right."""
    n = len(finals)
    k = n if k is None else k
    if not 1 <= k <= n:
        raise ValueError(f"k={k} out of range 1..{n}")
    out = None
    for alpha, final in zip(list(multipliers)[:k], finals[:k]):
        out = alpha * final if out is None else out + alpha * final
    return out


def group_forward(students: list[list[tuple[np.ndarray, np.ndarray]]], multipliers, classifier, x, k=None):
    """rep + classifier logits: distill.py:169-178 then :512. Returns (rep, logits)."""
    if classifier is None:
        raise ValueError("ensemble has no trained classifier")
    k = len(students) if k is None else k
    if not 1 <= k <= len(students):
        raise ValueError(f"k={k} out of range 1..{len(students)}")
    finals = [student_forward(s, x)[0] for s in students[:k]]
    rep = ensemble_rep(finals, multipliers, k)
    logits = dense_layer(classifier[0], classifier[1], rep, IDENTITY)
    return rep, logits


def predict(logits: np.ndarray) -> np.ndarray:
    """np.argmax over classes (distill.py:513); ties resolve to the lowest index."""
    return np.argmax(np.atleast_2d(logits), axis=1)


def group_forward_weights(w, x, k=None):
    """Convenience: run on a ``DenseGroupWeights`` container (its rounded, unpadded arrays)."""
    students = [w.student_layers(m) for m in range(w.n_students)]
    x = np.asarray(x, dtype=np.float64)
    return group_forward(students, [float(a) for a in w.alpha], w.classifier(), x, k)

"""Training-side evaluation on the engine.

The reference evaluates its ensemble during distillation and pruning with float64 numpy forwards
of every student (`distill.py`). These functions keep the reference's names, arguments and
results but take the student forward from the GPU (`StudentGroup`): one engine call yields
every student's final representation and the logits of every prefix k, which is all the
forward work of the reference's evaluation loops. Teacher-side quantities (the teacher's
representations and logits, `_teacher_reps` distill.py:285-287) are inputs: the teacher is the
distillation target, not a student.

Only the tiny reductions over [n, C] / [n, H] results happen on the host, as in the reference.
"""
from __future__ import annotations

import numpy as np

from .group import StudentGroup


def _softmax(z: np.ndarray) -> np.ndarray:
    """Row softmax with max shift (distill.py:433-436)."""
    z = z - z.max(axis=-1, keepdims=True)
    e = np.exp(z)
    return e / e.sum(axis=-1, keepdims=True)


def soft_cross_entropy(student_logits, teacher_logits, temperature: float = 1.0) -> float:
    """Cross-entropy of student logits against the teacher's soft labels (distill.py:439-452)."""
    if temperature <= 0:
        raise ValueError("temperature must be positive")
    s = np.asarray(student_logits, dtype=np.float64)
    t = np.asarray(teacher_logits, dtype=np.float64)
    if s.shape != t.shape:
        raise ValueError("logit width mismatch")
    if not (np.isfinite(s).all() and np.isfinite(t).all()):
        raise ValueError("logits must be finite")
    s, t = s / temperature, t / temperature
    log_p = s - s.max(axis=-1, keepdims=True)
    log_p = log_p - np.log(np.exp(log_p).sum(axis=-1, keepdims=True))
    return float(np.mean(np.sum(-_softmax(t) * log_p, axis=-1)))


def residual_mse(teacher_reps, group: StudentGroup, inputs, k: int | None = None) -> float:
    """Mean over samples of the half squared residual norm ||t - rep_k(x)||² / 2
    (distill.py:297-302); ``teacher_reps`` = teacher.forward(inputs)[0] (:285-287)."""
    t = np.asarray(teacher_reps, dtype=np.float64)
    prev = group.rep(inputs, k) if len(group) else np.zeros_like(t)
    prev = np.atleast_2d(prev)
    if prev.shape != np.atleast_2d(t).shape:
        raise ValueError(f"teacher reps {t.shape} do not match the ensemble's {prev.shape}")
    r = np.atleast_2d(t) - prev
    return 0.5 * float(np.mean(np.sum(r * r, axis=1)))


def prefix_objective(group: StudentGroup, xb, teacher_logits, temperature: float) -> tuple[float, np.ndarray]:
    """Value of the pruning objective on one batch — sum over k of the soft cross-entropy of
    prefix k against the teacher (the `total` of accumulate_prefix_gradients, distill.py:471-494)
    — plus the per-prefix terms. One engine forward serves all k."""
    _, prefix = group.finals_and_prefix_logits(xb)
    prefix = prefix.reshape(len(group), -1, prefix.shape[-1])
    terms = np.array([soft_cross_entropy(prefix[j], teacher_logits, temperature) for j in range(len(group))])
    total = 0.0
    for v in terms:  # left-to-right, as the reference accumulates `total`
        total += float(v)
    return total, terms


def prefix_accuracies(group: StudentGroup, inputs, labels) -> np.ndarray:
    """prefix_accuracy(state, data, k) for every k = 1..K (distill.py:508-513) from one forward."""
    _, prefix = group.finals_and_prefix_logits(inputs)
    prefix = prefix.reshape(len(group), -1, prefix.shape[-1])
    y = np.asarray(labels)
    return np.array([float(np.mean(np.argmax(prefix[j], axis=1) == y)) for j in range(len(group))])


def ensemble_accuracy_via_teacher_head(head_weight, head_bias, group: StudentGroup, inputs, labels) -> float:
    """Accuracy of the full ensemble representation pushed through the teacher's head
    (distill.py:676-683): logits = W_head · rep(x) + b_head (nnkernel.py:73, identity)."""
    rep = np.atleast_2d(group.rep(inputs))
    w = np.asarray(head_weight, dtype=np.float64)
    b = np.asarray(head_bias, dtype=np.float64)
    if w.shape[1] != rep.shape[1]:
        raise ValueError(f"input width {rep.shape[1]} does not match layer in_dim {w.shape[1]}")
    logits = rep @ w.T + b
    return float(np.mean(np.argmax(logits, axis=1) == np.asarray(labels)))

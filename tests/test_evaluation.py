"""Training-side evaluation: `paper_2408_12526_b200.evaluation` over the engine.

CPU: the host-side restatements (soft cross-entropy, prefix objective, residual MSE, teacher-head
accuracy) run over the float64 oracle's finals reproduce the reference's own numbers for the
reference-trained checkpoint (tests/golden/training_eval_ref.npz, made by make_golden.py).
GPU: the same functions over one engine forward (sp_group_forward_dense_eval / _eval) agree with
the reference and with the oracle on identical rounded weights.
"""
import json

import numpy as np
import pytest

from goldens import GOLDEN
from paper_2408_12526_b200 import evaluation as ev
from paper_2408_12526_b200.checkpoint import ensemble_arrays_from_dict

REF = np.load(GOLDEN / "training_eval_ref.npz")


class OracleEnsemble:
    """The duck-typed surface evaluation.py uses (len, rep, finals_and_prefix_logits) on the float64
    oracle — test infrastructure only."""

    def __init__(self, students, alphas, clf):
        self.students, self.alphas, self.clf = students, alphas, clf

    def __len__(self):
        return len(self.students)

    def rep(self, x, k=None):
        from oracle.dense import group_forward

        return group_forward(self.students, self.alphas, self.clf, x, k)[0]

    def finals_and_prefix_logits(self, x, k=None):
        from oracle.dense import dense_layer, ensemble_rep, student_forward

        finals = [student_forward(s, x)[0] for s in self.students]
        prefix = [dense_layer(self.clf[0], self.clf[1], ensemble_rep(finals, self.alphas, j), "identity")
                  for j in range(1, len(finals) + 1)]
        return np.stack(finals), np.stack(prefix)


def _oracle_trained():
    d = json.loads((GOLDEN / "ensemble_trained.json").read_text())
    return OracleEnsemble(*ensemble_arrays_from_dict(d))


def test_soft_cross_entropy_restatement():
    rng = np.random.default_rng(0)
    s, t = rng.normal(size=(7, 3)), rng.normal(size=(7, 3))
    p = np.exp(t / 2.0) / np.exp(t / 2.0).sum(1, keepdims=True)
    ls = s / 2.0 - np.log(np.exp(s / 2.0).sum(1, keepdims=True))
    assert ev.soft_cross_entropy(s, t, 2.0) == pytest.approx(float(np.mean(-(p * ls).sum(1))), rel=1e-13)
    with pytest.raises(ValueError):
        ev.soft_cross_entropy(s, t, 0.0)
    with pytest.raises(ValueError):
        ev.soft_cross_entropy(s, t[:, :2])
    with pytest.raises(ValueError):
        ev.soft_cross_entropy(s * np.inf, t)


def test_evaluation_restatements_match_reference_on_oracle():
    g = _oracle_trained()
    x, y = REF["x_val"], REF["y_val"]
    for k in range(1, len(g) + 1):
        assert ev.residual_mse(REF["teacher_rep"], g, x, k) == pytest.approx(REF["residual_mse"][k - 1], rel=1e-12)
    for temp in (1.0, 2.0):
        total, terms = ev.prefix_objective(g, x, REF["teacher_logits"], temp)
        assert total == pytest.approx(float(REF[f"prefix_total_T{temp:g}"]), rel=1e-12)
        assert len(terms) == len(g)
    acc = ev.ensemble_accuracy_via_teacher_head(REF["head_w"], REF["head_b"], g, x, y)
    assert acc == float(REF["acc_teacher_head"])
    task = np.load(GOLDEN / "ensemble_trained_task.npz")
    np.testing.assert_array_equal(ev.prefix_accuracies(g, task["x_val"], task["y_val"]), task["acc_val"])


@pytest.mark.reference
def test_evaluation_restatements_match_live_reference():
    import sys

    sys.path.insert(0, "/root/reference/pkg/src")
    from studentpar import distill as dst

    rng = np.random.default_rng(3)
    for temp in (0.5, 1.0, 4.0):
        s, t = rng.normal(size=(11, 4)), rng.normal(size=(11, 4))
        assert ev.soft_cross_entropy(s, t, temp) == dst.soft_cross_entropy(s, t, temp)


@pytest.mark.gpu
def test_engine_training_eval_matches_reference_checkpoint():
    from paper_2408_12526_b200 import StudentGroup

    grp = StudentGroup.from_checkpoint(GOLDEN / "ensemble_trained.json", max_tokens=256)
    x, y = REF["x_val"], REF["y_val"]
    # reference weights are float64; the engine rounds matrices to fp16 (same bound as the logits test)
    for k in range(1, len(grp) + 1):
        assert ev.residual_mse(REF["teacher_rep"], grp, x, k) == pytest.approx(REF["residual_mse"][k - 1], rel=5e-3)
    for temp in (1.0, 2.0):
        total, _ = ev.prefix_objective(grp, x, REF["teacher_logits"], temp)
        assert total == pytest.approx(float(REF[f"prefix_total_T{temp:g}"]), rel=5e-3)
    assert ev.ensemble_accuracy_via_teacher_head(REF["head_w"], REF["head_b"], grp, x, y) == float(REF["acc_teacher_head"])
    task = np.load(GOLDEN / "ensemble_trained_task.npz")
    np.testing.assert_array_equal(ev.prefix_accuracies(grp, task["x_val"], task["y_val"]), task["acc_val"])
    np.testing.assert_array_equal(ev.prefix_accuracies(grp, task["x_test"], task["y_test"]), task["acc_test"])


@pytest.mark.gpu
def test_engine_finals_and_prefix_logits_match_oracle_dense():
    """Identical rounded weights: every student's final and every prefix's logits vs the oracle."""
    from oracle.dense import group_forward_weights
    from paper_2408_12526_b200 import StudentGroup, random_dense_group

    w = random_dense_group(d_in=64, rep_dim=256, depth=2, n_students=5, n_classes=3, seed=9)
    grp = StudentGroup(w, max_tokens=512)
    x = np.random.default_rng(1).normal(size=(200, 64))
    xr = np.float16(x).astype(np.float64)
    finals, prefix = grp.finals_and_prefix_logits(x)
    assert finals.shape == (5, 200, 256) and prefix.shape == (5, 200, 3)
    from oracle.dense import student_forward

    for m in range(5):
        ref = student_forward(w.student_layers(m), xr)[0]
        assert np.abs(finals[m] - ref).max() <= 2e-3  # tanh outputs, |S| <= 1
    for k in range(1, 6):
        _, z_ref = group_forward_weights(w, xr, k)
        assert np.abs(prefix[k - 1] - z_ref).max() <= 1e-3 * np.abs(z_ref).max()
        np.testing.assert_allclose(prefix[k - 1], grp.logits(x, k), rtol=0, atol=1e-5)
    f1, z1 = grp.finals_and_prefix_logits(x[0])  # 1-D input: sample axis dropped
    assert f1.shape == (5, 256) and z1.shape == (5, 3)
    fk, zk = grp.finals_and_prefix_logits(x, k=2)
    assert fk.shape == (2, 200, 256) and zk.shape == (2, 200, 3)


@pytest.mark.gpu
def test_engine_finals_and_prefix_logits_match_oracle_bert():
    from oracle.bert import OracleBertGroup
    from paper_2408_12526_b200 import PRESETS, StudentGroup, random_bert_group

    cfg, _ = PRESETS["tiny"]
    w = random_bert_group(cfg, 4, seed=3)
    grp = StudentGroup(w, max_tokens=512, max_seqs=8)
    orc = OracleBertGroup(w)
    rng = np.random.default_rng(5)
    seqs = [np.r_[101, rng.integers(1000, cfg.vocab, size=L - 1)].astype(np.int32) for L in (1, 9, 33, 64)]
    finals, prefix = grp.finals_and_prefix_logits(seqs)
    assert finals.shape == (4, 4, cfg.hidden) and prefix.shape == (4, 4, 2)
    for k in range(1, 5):
        _, z_ref = orc.forward(seqs, k)
        assert np.abs(prefix[k - 1] - z_ref).max() <= 1e-3 * np.abs(z_ref).max()
    for m in range(4):
        ref = orc.pooled(m, seqs)
        assert np.abs(finals[m] - ref).max() <= 2e-3

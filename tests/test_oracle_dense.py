"""The float64 oracle's dense-student group vs the reference (CPU).

Pinned three ways: (1) the reference's own known-answer tests restated (test_nnkernel.py:51-67,
:140-155; test_distill.py:59-94), (2) the committed golden vectors produced by the unmodified
reference (tests/golden/make_golden.py), (3) the live reference package when it is importable.
"""
import math

import numpy as np
import pytest

from goldens import DENSE_CASES, load_dense
from oracle import dense as od


def scalar_dense(weight, bias, x, act):
    """Independent scalar loop, as test_nnkernel.py:17-25."""
    out = []
    for i in range(weight.shape[0]):
        acc = bias[i]
        for j in range(weight.shape[1]):
            acc += weight[i][j] * x[j]
        out.append(math.tanh(acc) if act == od.TANH else acc)
    return np.array(out)


def test_identity_layer_kat():  # test_nnkernel.py:51-53
    assert np.array_equal(od.dense_layer(np.eye(2), np.zeros(2), np.array([3.0, -1.0]), od.IDENTITY), [3.0, -1.0])


def test_zero_weight_tanh_kat():  # test_nnkernel.py:56-59
    out = od.dense_layer(np.zeros((2, 2)), np.ones(2), np.array([5.0, 5.0]), od.TANH)
    assert np.allclose(out, [math.tanh(1.0)] * 2, rtol=0, atol=0)


def test_dense_matches_scalar_oracle():  # test_nnkernel.py:62-67
    rng = np.random.default_rng(1)
    w, b, x = rng.normal(size=(3, 2)), rng.normal(size=3), rng.normal(size=2)
    np.testing.assert_allclose(od.dense_layer(w, b, x, od.TANH), scalar_dense(w, b, x, od.TANH), rtol=1e-15)


def test_dense_width_mismatch_raises():  # test_nnkernel.py:70-73
    with pytest.raises(ValueError):
        od.dense_layer(np.eye(2), np.zeros(2), np.zeros(3), od.IDENTITY)


def _constant_student(d_in, rep_dim, value):  # test_distill.py:16-21
    z = np.zeros
    return [(z((rep_dim, d_in)), z(rep_dim)), (z((rep_dim, rep_dim)), z(rep_dim)),
            (z((rep_dim, rep_dim)), np.arctanh(np.asarray(value, dtype=float)))]


def test_ensemble_weighted_sum_kat():  # test_distill.py:59-69 (tanh students; bias = atanh(value))
    s0 = _constant_student(3, 2, [0.5, 0.0])
    s1 = _constant_student(3, 2, [0.0, 0.5])
    finals = [od.student_forward(s, np.zeros(3))[0] for s in (s0, s1)]
    np.testing.assert_allclose(od.ensemble_rep(finals, [1.0, 0.5], 2), [0.5, 0.25], rtol=1e-15)
    np.testing.assert_allclose(od.ensemble_rep(finals, [1.0, 0.5], 1), [0.5, 0.0], rtol=1e-15)


def test_ensemble_scalar_loop_kat():  # test_distill.py:72-83, alphas [1, 0.7, -0.4]
    rng = np.random.default_rng(1)
    students = []
    for _ in range(3):
        dims = [(4, 3), (4, 4), (4, 4)]
        students.append([(rng.uniform(-0.9, 0.9, d), rng.normal(size=d[0])) for d in dims])
    alphas = [1.0, 0.7, -0.4]
    x = rng.normal(size=3)
    expected = np.zeros(4)
    for a, s in zip(alphas, students):
        h = x
        for w, b in s:
            h = scalar_dense(w, b, h, od.TANH)
        expected += a * h
    finals = [od.student_forward(s, x)[0] for s in students]
    np.testing.assert_allclose(od.ensemble_rep(finals, alphas, 3), expected, rtol=1e-12)


def test_k_out_of_range_raises():  # test_distill.py:86-89
    with pytest.raises(ValueError):
        od.ensemble_rep([np.ones(2)], [1.0], 2)
    with pytest.raises(ValueError):
        od.ensemble_rep([np.ones(2)], [1.0], 0)


def test_student_needs_two_layers():  # nnkernel.py:265-266
    with pytest.raises(ValueError):
        od.student_forward([(np.eye(2), np.zeros(2)), (np.eye(2), np.zeros(2))], np.zeros(2))


def test_mid_tap_is_ceil_half():  # nnkernel.py:280-283, test_nnkernel.py:133-155
    rng = np.random.default_rng(3)
    for depth in range(2, 7):
        layers = [(rng.normal(size=(3, 2)), rng.normal(size=3))] + [(rng.normal(size=(3, 3)), rng.normal(size=3))
                                                                    for _ in range(depth)]
        x = rng.normal(size=2)
        h = od.dense_layer(*layers[0], x)
        taps = []
        for w, b in layers[1:]:
            h = od.dense_layer(w, b, h)
            taps.append(h)
        _, mid = od.student_forward(layers, x)
        np.testing.assert_array_equal(mid, taps[(depth + 1) // 2 - 1])


@pytest.mark.parametrize("name", DENSE_CASES)
def test_oracle_matches_reference_golden(name):
    """Bit-level agreement with the reference's outputs (same float64 algorithm, same order)."""
    case = load_dense(name)
    for k in range(1, case["K"] + 1):
        rep, logits = od.group_forward(case["students"], case["alphas"], case["classifier"], case["x"], k)
        np.testing.assert_allclose(rep, case["rep"][k], rtol=1e-12, atol=1e-14)
        np.testing.assert_allclose(logits, case["logits"][k], rtol=1e-12, atol=1e-14)
        assert np.array_equal(od.predict(logits), case["pred"][k])
        rep1, _ = od.group_forward(case["students"], case["alphas"], case["classifier"], case["x"][0], k)
        np.testing.assert_allclose(rep1, case["rep1"][k], rtol=1e-12, atol=1e-14)
    _, mid = od.student_forward(case["students"][0], case["x"])
    np.testing.assert_allclose(mid, case["mid0"], rtol=1e-12, atol=1e-14)


@pytest.mark.reference
def test_oracle_matches_live_reference(ref):
    """Against the reference package itself on fresh random groups (build container only)."""
    rng = np.random.Generator(np.random.PCG64(42))
    for d_in, rep_dim, depth, K in [(5, 7, 2, 3), (16, 32, 3, 4)]:
        students = [ref.nn.StudentModel.build(d_in, rep_dim, depth, rng) for _ in range(K)]
        alphas = [1.0] + list(rng.uniform(-1, 1, size=K - 1))
        clf = ref.nn.DenseLayer.init(3, rep_dim, ref.nn.IDENTITY, rng)
        state = ref.distill.EnsembleState(students, alphas, clf)
        x = rng.normal(size=(11, d_in))
        layers = [[(s.input_proj.weight, s.input_proj.bias)] + [(l.weight, l.bias) for l in s.layers]
                  for s in students]
        for k in range(1, K + 1):
            rep, logits = od.group_forward(layers, alphas, (clf.weight, clf.bias), x, k)
            np.testing.assert_array_equal(rep, state.rep(x, k))
            np.testing.assert_array_equal(logits, clf.forward(state.rep(x, k)))


def test_weights_container_roundtrip_matches_golden():
    """paper_2408_12526_b200.weights (padding to the engine's tile multiples) keeps the logical
    group exact: the oracle on the padded container's unpadded view equals the golden."""
    from paper_2408_12526_b200.weights import dense_group_from_arrays

    case = load_dense("pad")  # engine-precision fixture: rounding is the identity here
    w = dense_group_from_arrays(case["students"], case["alphas"], case["classifier"])
    assert w.hidden_padded == 256 and w.d_in_padded == 128
    for k in range(1, case["K"] + 1):
        rep, logits = od.group_forward_weights(w, case["x"], k)
        np.testing.assert_allclose(logits, case["logits"][k], rtol=1e-12, atol=1e-14)


def test_weight_lo_terms_carry_float64_checkpoints():
    """Float64 reference weights travel as fp16 (hi, lo) pairs (ABI v3): the group's represented
    weights reproduce the reference's own logits to ~1e-6 on the reference-trained checkpoint and
    the 'tiny' golden, where fp16 weights alone are 1e-3..3e-2 off. fp16-exact sources and
    exact=False carry no lo terms; subset() keeps them aligned with the students."""
    from conftest import rel_err_rows
    from goldens import GOLDEN, load_trained_task
    from paper_2408_12526_b200.checkpoint import load_ensemble_weights
    from paper_2408_12526_b200.weights import dense_group_from_arrays

    task = load_trained_task()
    w = load_ensemble_weights(GOLDEN / "ensemble_trained.json")
    assert w.exact_weights and w.w_in_lo.dtype == np.float16 and w.w_layers_lo.shape == w.w_layers.shape
    for k in range(1, len(w.alpha) + 1):
        _, z = od.group_forward_weights(w, task["x_val"], k)
        assert rel_err_rows(z, task[f"logits_val_k{k}"]) <= 1e-5
    case = load_dense("tiny")
    for exact, bound in ((True, 1e-5), (False, 1e-2)):
        wt = dense_group_from_arrays(case["students"], case["alphas"], case["classifier"], exact=exact)
        assert wt.exact_weights == exact
        err = max(rel_err_rows(od.group_forward_weights(wt, case["x"], k)[1], case["logits"][k])
                  for k in range(1, case["K"] + 1))
        assert err <= bound
    pad = load_dense("pad")  # engine-precision fixture: weights already fp16 values
    assert not dense_group_from_arrays(pad["students"], pad["alphas"], pad["classifier"]).exact_weights
    sub = w.subset([2, 0])
    np.testing.assert_array_equal(sub.w_layers_lo[:, 0], w.w_layers_lo[:, 2])
    np.testing.assert_array_equal(sub.w_in_lo[1], w.w_in_lo[0])

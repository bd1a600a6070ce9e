"""Known-answer tests that pin the oracle's BERT-student pieces (CPU).

The reference has no embedding / attention / LayerNorm / GELU code, so these four
pieces are pinned by closed forms: attention with one key returns V, identical keys
average V, LayerNorm of a constant row is beta, GELU(0) = 0 and GELU(x) -> x, a student whose
encoder layers are all zero reduces to pooler(LN(embedding)), and packed sequences never leak into
each other. Every affine map inside the student is the pinned oracle.dense.dense_layer.
"""
import math

import numpy as np
import pytest

from oracle import bert as ob
from oracle.dense import dense_layer
from paper_2408_12526_b200.weights import BertConfig, random_bert_group

SMALL = BertConfig(hidden=16, n_layers=2, n_heads=2, vocab=64, max_pos=24, n_classes=3)


@pytest.fixture(scope="module")
def small_group():
    return random_bert_group(SMALL, 3, seed=5)


def test_layer_norm_constant_row_is_beta():
    beta = np.arange(6.0)
    out = ob.layer_norm(np.full((2, 6), 3.5), np.ones(6) * 2.0, beta, 1e-12)  # exact mean
    np.testing.assert_allclose(out, np.stack([beta, beta]), atol=1e-12)


def test_layer_norm_standardizes():
    x = np.random.default_rng(0).normal(3.0, 5.0, size=(4, 32))
    y = ob.layer_norm(x, np.ones(32), np.zeros(32), 1e-12)
    np.testing.assert_allclose(y.mean(axis=1), 0.0, atol=1e-12)
    np.testing.assert_allclose(y.var(axis=1), 1.0, atol=1e-9)


def test_gelu_known_values():
    assert ob.gelu(np.array(0.0)) == 0.0
    np.testing.assert_allclose(ob.gelu(np.array(1.0)), 0.8413447460685429, rtol=1e-15)  # Phi(1)
    np.testing.assert_allclose(ob.gelu(np.array(-1.0)), -0.15865525393145707, rtol=1e-14)
    np.testing.assert_allclose(ob.gelu(np.array(12.0)), 12.0, rtol=1e-15)
    assert abs(ob.gelu(np.array(-12.0))) < 1e-30


def test_attention_single_key_returns_v():
    rng = np.random.default_rng(1)
    q, k, v = rng.normal(size=(1, 3, 4)), rng.normal(size=(1, 3, 4)), rng.normal(size=(1, 3, 4))
    np.testing.assert_allclose(ob.attention(q, k, v), v, rtol=1e-15)


def test_attention_identical_keys_average_values():
    rng = np.random.default_rng(2)
    L = 5
    q = rng.normal(size=(L, 2, 8))
    k = np.repeat(rng.normal(size=(1, 2, 8)), L, axis=0)
    v = rng.normal(size=(L, 2, 8))
    np.testing.assert_allclose(ob.attention(q, k, v), np.repeat(v.mean(axis=0, keepdims=True), L, axis=0),
                               rtol=1e-13)


def test_attention_matches_scalar_loops():
    rng = np.random.default_rng(3)
    L, h, d = 6, 2, 4
    q, k, v = (rng.normal(size=(L, h, d)) for _ in range(3))
    out = np.zeros((L, h, d))
    for hh in range(h):
        for i in range(L):
            s = [sum(q[i, hh, c] * k[j, hh, c] for c in range(d)) / math.sqrt(d) for j in range(L)]
            mx = max(s)
            p = [math.exp(x - mx) for x in s]
            z = sum(p)
            for c in range(d):
                out[i, hh, c] = sum(p[j] / z * v[j, hh, c] for j in range(L))
    np.testing.assert_allclose(ob.attention(q, k, v), out, rtol=1e-12)


def test_zero_encoder_reduces_to_pooled_layernormed_embedding():
    w = random_bert_group(SMALL, 1, seed=6)  # own copy: mutated below
    for name in ["w_qkv", "b_qkv", "w_o", "b_o", "w_ffn1", "b_ffn1", "w_ffn2", "b_ffn2"]:
        getattr(w, name)[...] = 0
    w.ln1_gamma[...] = 1
    w.ln1_beta[...] = 0
    w.ln2_gamma[...] = 1
    w.ln2_beta[...] = 0
    w.emb_ln_gamma[...] = 1
    w.emb_ln_beta[...] = 0
    orc = ob.OracleBertGroup(w)
    ids = np.array([3, 17, 40, 9], np.int32)
    e = (w.word_emb[0][ids].astype(np.float64) + w.pos_emb[0][:4].astype(np.float64)
         + w.type_emb[0].astype(np.float64))
    h = ob.layer_norm(e, 1.0, 0.0, SMALL.ln_eps)
    for _ in range(2 * SMALL.n_layers):  # each residual sub-block adds exact zeros, then LN again
        h = ob.layer_norm(h, 1.0, 0.0, SMALL.ln_eps)
    expected = dense_layer(w.w_pool[0].astype(np.float64), w.b_pool[0].astype(np.float64), h[0])
    np.testing.assert_allclose(orc.pooled(0, [ids])[0], expected, rtol=1e-12, atol=1e-14)


def test_packed_sequences_do_not_leak(small_group):
    orc = ob.OracleBertGroup(small_group)
    a = np.array([1, 5, 9, 2, 33], np.int32)
    b1 = np.array([7, 8], np.int32)
    b2 = np.array([60, 61, 62], np.int32)
    rep_ab1, _ = orc.forward([a, b1])
    rep_ab2, _ = orc.forward([a, b2])
    rep_a, _ = orc.forward([a])
    # (BLAS may reorder sums by batch shape: agreement to rounding, not bitwise)
    np.testing.assert_allclose(rep_ab1[0], rep_ab2[0], rtol=1e-13, atol=1e-15)
    np.testing.assert_allclose(rep_ab1[0], rep_a[0], rtol=1e-13, atol=1e-15)
    # positions restart at 0 for each packed sequence
    rep_b1_alone, _ = orc.forward([b1])
    np.testing.assert_allclose(rep_ab1[1], rep_b1_alone[0], rtol=1e-13, atol=1e-15)
    ids = np.concatenate([a, b1])
    cu = np.array([0, 5, 7])
    rep_p, z_p = orc.forward_packed(ids, cu)
    np.testing.assert_array_equal(rep_p, rep_ab1)


def test_prefix_k_is_alpha_weighted_sum(small_group):
    orc = ob.OracleBertGroup(small_group)
    seqs = [np.array([4, 5, 6], np.int32), np.array([9], np.int32)]
    pooled = [orc.pooled(m, seqs) for m in range(3)]
    for k in (1, 2, 3):
        rep, z = orc.forward(seqs, k)
        exp = sum(orc.alpha[m] * pooled[m] for m in range(k))
        np.testing.assert_allclose(rep, exp, rtol=1e-14)
        np.testing.assert_allclose(z, rep @ orc.w_cls.T + orc.b_cls, rtol=1e-14)
    assert orc.alpha[0] == 1.0


def test_input_errors(small_group):
    orc = ob.OracleBertGroup(small_group)
    with pytest.raises(ValueError):
        orc.forward([np.array([], np.int32)])
    with pytest.raises(ValueError):
        orc.forward([np.array([64], np.int32)])
    with pytest.raises(ValueError):
        orc.forward([np.zeros(25, np.int32)])
    with pytest.raises(ValueError):
        orc.forward([np.array([1], np.int32)], k=4)

"""Float64 restatement of the BERT-style student group — TEST INFRASTRUCTURE (oracle/__init__.py).

The reference artifact never implements a transformer student, so this
file restates the paper's students from PAPER.md and standard BERT semantics:

* residual post-LN encoder layers (PAPER.md:853-859; BERT-2L students PAPER.md:1297, :1733),
* the student's output is its final pooled representation =
  tanh(W_p h_CLS + b_p), a reference ``DenseLayer(H, H, tanh)`` (nnkernel.py:66-76),
* the group output is the boosting sum of the first k students' representations through the
  shared classifier (PAPER.md:878-882 Eq. 1; EnsembleState.rep distill.py:169-178, :512).

Builder decisions: erf-exact GELU, LayerNorm eps from the config (1e-12, BERT),
token type 0 for every token, positions restart at 0 for every packed sequence, no padding and no
attention mask beyond each sequence's own tokens. These four pieces — embedding gather, LayerNorm,
GELU, attention — are "parity unpinned" by the reference; tests/test_oracle_bert.py pins them with
closed-form known-answer tests.
"""
from __future__ import annotations

import numpy as np
from scipy.special import erf

from .dense import IDENTITY, TANH, dense_layer, ensemble_rep


def layer_norm(x: np.ndarray, gamma: np.ndarray, beta: np.ndarray, eps: float) -> np.ndarray:
    """(x - mean) / sqrt(var + eps) * gamma + beta over the last axis, biased variance (BERT)."""
    mean = x.mean(axis=-1, keepdims=True)
    var = ((x - mean) ** 2).mean(axis=-1, keepdims=True)
    return (x - mean) / np.sqrt(var + eps) * gamma + beta


def gelu(x: np.ndarray) -> np.ndarray:
    """Exact (erf) GELU: 0.5 x (1 + erf(x / sqrt 2))."""
    return 0.5 * x * (1.0 + erf(x / np.sqrt(2.0)))


def attention(q: np.ndarray, k: np.ndarray, v: np.ndarray) -> np.ndarray:
    """Unmasked softmax(Q K^T / sqrt(d)) V for one sequence; q, k, v: [L, heads, d] -> [L, heads, d]."""
    d = q.shape[-1]
    s = np.einsum("qhd,khd->hqk", q, k) / np.sqrt(d)
    s = s - s.max(axis=-1, keepdims=True)
    p = np.exp(s)
    p /= p.sum(axis=-1, keepdims=True)
    return np.einsum("hqk,khd->qhd", p, v)


def split_ids(ids: np.ndarray, cu_seqlens: np.ndarray) -> list[np.ndarray]:
    cu = np.asarray(cu_seqlens, dtype=np.int64)
    return [np.asarray(ids[cu[b]:cu[b + 1]]) for b in range(len(cu) - 1)]


class OracleBertGroup:
    """Float64 copy of a ``BertGroupWeights`` (the same fp16/fp32-rounded values the engine uses)."""

    def __init__(self, w):
        self.cfg = w.cfg
        self.w = w
        self.alpha = [float(a) for a in w.alpha]
        self.w_cls = w.w_cls.astype(np.float64)
        self.b_cls = w.b_cls.astype(np.float64)
        self._cache: dict[int, dict] = {}

    @property
    def n_students(self) -> int:
        return len(self.alpha)

    def student(self, m: int) -> dict:
        if m not in self._cache:
            w, f = self.w, np.float64
            layers = []
            for l in range(self.cfg.n_layers):
                layers.append(dict(
                    qkv=(w.w_qkv[l, m].astype(f), w.b_qkv[l, m].astype(f)),
                    o=(w.w_o[l, m].astype(f), w.b_o[l, m].astype(f)),
                    ln1=(w.ln1_gamma[l, m].astype(f), w.ln1_beta[l, m].astype(f)),
                    ffn1=(w.w_ffn1[l, m].astype(f), w.b_ffn1[l, m].astype(f)),
                    ffn2=(w.w_ffn2[l, m].astype(f), w.b_ffn2[l, m].astype(f)),
                    ln2=(w.ln2_gamma[l, m].astype(f), w.ln2_beta[l, m].astype(f)),
                ))
            self._cache[m] = dict(
                word=w.word_emb[m], pos=w.pos_emb[m], type=w.type_emb[m].astype(f),
                emb_ln=(w.emb_ln_gamma[m].astype(f), w.emb_ln_beta[m].astype(f)),
                layers=layers, pool=(w.w_pool[m].astype(f), w.b_pool[m].astype(f)),
            )
        return self._cache[m]

    def encode(self, m: int, ids: np.ndarray) -> np.ndarray:
        """One student on one unpadded sequence -> final hidden states [L, H]."""
        cfg, s = self.cfg, self.student(m)
        L = len(ids)
        if L < 1:
            raise ValueError("empty sequence")
        if L > cfg.max_pos:
            raise ValueError(f"sequence of {L} tokens exceeds max_pos {cfg.max_pos}")
        ids = np.asarray(ids, dtype=np.int64)
        if ids.min() < 0 or ids.max() >= cfg.vocab:
            raise ValueError("token id outside vocab")
        x = s["word"][ids].astype(np.float64) + s["pos"][:L].astype(np.float64) + s["type"]
        x = layer_norm(x, *s["emb_ln"], cfg.ln_eps)
        nh, hd, H = cfg.n_heads, cfg.head_dim, cfg.hidden
        for lay in s["layers"]:
            qkv = dense_layer(*lay["qkv"], x, IDENTITY)
            q = qkv[:, :H].reshape(L, nh, hd)
            k = qkv[:, H:2 * H].reshape(L, nh, hd)
            v = qkv[:, 2 * H:].reshape(L, nh, hd)
            ctx = attention(q, k, v).reshape(L, H)
            x = layer_norm(x + dense_layer(*lay["o"], ctx, IDENTITY), *lay["ln1"], cfg.ln_eps)
            f = gelu(dense_layer(*lay["ffn1"], x, IDENTITY))
            x = layer_norm(x + dense_layer(*lay["ffn2"], f, IDENTITY), *lay["ln2"], cfg.ln_eps)
        return x

    def pooled(self, m: int, seqs: list[np.ndarray]) -> np.ndarray:
        """Student m's final pooled representation per sequence: tanh(W_p h_CLS + b_p) -> [B, H]."""
        cls = np.stack([self.encode(m, ids)[0] for ids in seqs])
        return dense_layer(*self.student(m)["pool"], cls, TANH)

    def forward(self, seqs: list[np.ndarray], k: int | None = None, students=None):
        """(rep, logits) of the prefix-k group: rep = sum_{m<k} alpha_m pooled_m; logits = W_c rep + b_c."""
        n = self.n_students
        k = n if k is None else k
        if not 1 <= k <= n:
            raise ValueError(f"k={k} out of range 1..{n}")
        finals = [self.pooled(m, seqs) for m in range(k)]
        rep = ensemble_rep(finals, self.alpha, k)
        return rep, dense_layer(self.w_cls, self.b_cls, rep, IDENTITY)

    def forward_packed(self, ids: np.ndarray, cu_seqlens: np.ndarray, k: int | None = None):
        return self.forward(split_ids(ids, cu_seqlens), k)

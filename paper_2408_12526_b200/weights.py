"""Host-side student-group weights: configs, seeded random init, reference-ensemble import, packing.

Two student kinds share one group head (boosting sum + shared classifier, distill.py:139-178):

* ``dense`` — the reference's own ``StudentModel`` (nnkernel.py:256-301): tanh(input_proj) followed
  by ``depth`` tanh H x H layers. Imported from a reference ``EnsembleState`` (or an
  ``ensemble-checkpoint-v1`` file) so parity is pinned by the reference itself.
* ``bert`` — the paper's BERT-style flat student: word+position+type
  embeddings with LayerNorm, ``n_layers`` post-LN encoder layers (QKV, attention, O + residual + LN,
  FFN1 + GELU, FFN2 + residual + LN) and a tanh pooler on the CLS row; every affine map is a
  reference ``DenseLayer`` in (out, in) layout.

"Identical weights" (BASELINE.json north star): matrices are rounded to fp16 and vectors
(biases, LayerNorm, alpha, classifier) to fp32 ONCE here; the CUDA engine and the float64 oracle
both consume exactly these rounded values.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field, replace

import numpy as np

from .seeding import rng_for


# --------------------------------------------------------------------------- configs
@dataclass(frozen=True)
class BertConfig:
    hidden: int = 768
    n_layers: int = 2
    n_heads: int = 12
    ffn: int = 0  # 0 -> 4 * hidden
    vocab: int = 30522
    max_pos: int = 512
    n_classes: int = 2
    ln_eps: float = 1e-12

    def __post_init__(self):
        if self.ffn == 0:
            object.__setattr__(self, "ffn", 4 * self.hidden)
        if self.hidden % self.n_heads:
            raise ValueError("hidden must be divisible by n_heads")

    @property
    def head_dim(self) -> int:
        return self.hidden // self.n_heads


# BASELINE.json configs: tiny (K=4, H=128, 4 heads), BERT-base-sized (K=8, H=768, 12 heads),
# BERT-large-sized (K=12, H=1024, 16 heads), K=32 at H=768. All: 2 layers, F = 4H, C = 2.
PRESETS: dict[str, tuple[BertConfig, int]] = {
    "tiny": (BertConfig(hidden=128, n_heads=4), 4),
    "base": (BertConfig(hidden=768, n_heads=12), 8),
    "large": (BertConfig(hidden=1024, n_heads=16), 12),
    "k32": (BertConfig(hidden=768, n_heads=12), 32),
}


def _f16(a: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float16)


def _f32(a: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


# --------------------------------------------------------------------------- BERT kind
@dataclass
class BertGroupWeights:
    """Student-stacked BERT-kind weights (leading axes [n_layers][K] or [K])."""

    cfg: BertConfig
    word_emb: np.ndarray      # f16 [K, V, H]
    pos_emb: np.ndarray       # f16 [K, P, H]
    type_emb: np.ndarray      # f16 [K, H]
    emb_ln_gamma: np.ndarray  # f32 [K, H]
    emb_ln_beta: np.ndarray
    w_qkv: np.ndarray         # f16 [NL, K, 3H, H]
    b_qkv: np.ndarray         # f32 [NL, K, 3H]
    w_o: np.ndarray           # f16 [NL, K, H, H]
    b_o: np.ndarray
    ln1_gamma: np.ndarray
    ln1_beta: np.ndarray
    w_ffn1: np.ndarray        # f16 [NL, K, F, H]
    b_ffn1: np.ndarray
    w_ffn2: np.ndarray        # f16 [NL, K, H, F]
    b_ffn2: np.ndarray
    ln2_gamma: np.ndarray
    ln2_beta: np.ndarray
    w_pool: np.ndarray        # f16 [K, H, H]
    b_pool: np.ndarray        # f32 [K, H]
    alpha: np.ndarray         # f32 [K], alpha[0] == 1 (distill.py:152-153)
    w_cls: np.ndarray         # f32 [C, H]
    b_cls: np.ndarray         # f32 [C]
    kind: str = field(default="bert", init=False)

    @property
    def n_students(self) -> int:
        return int(self.alpha.shape[0])

    def subset(self, idx) -> "BertGroupWeights":
        """Weights of the students ``idx`` (in that order); the classifier is shared."""
        idx = np.asarray(idx, dtype=np.int64)
        per_student = dict(word_emb=0, pos_emb=0, type_emb=0, emb_ln_gamma=0, emb_ln_beta=0, w_pool=0, b_pool=0,
                           alpha=0)
        per_layer = ["w_qkv", "b_qkv", "w_o", "b_o", "ln1_gamma", "ln1_beta", "w_ffn1", "b_ffn1", "w_ffn2",
                     "b_ffn2", "ln2_gamma", "ln2_beta"]
        kw = {}
        for name in per_student:
            kw[name] = np.ascontiguousarray(getattr(self, name)[idx])
        for name in per_layer:
            kw[name] = np.ascontiguousarray(getattr(self, name)[:, idx])
        return BertGroupWeights(cfg=self.cfg, w_cls=self.w_cls, b_cls=self.b_cls, **kw)


def _alpha_draw(seed: int, k: int) -> np.ndarray:
    """alpha = [1] + U(0.2, 1.0)^(K-1); alpha_0 pinned to 1 as in distill.py:152-153."""
    rng = rng_for(seed, "alpha")
    return _f32(np.concatenate([[1.0], rng.uniform(0.2, 1.0, size=k - 1)]))


def random_bert_group(cfg: BertConfig, n_students: int, seed: int = 0, students=None) -> BertGroupWeights:
    """Seeded random-init BERT-kind group: matrices N(0, 0.02) (BERT init), small random biases and
    LayerNorm perturbations (so bias/LN bugs cannot hide behind zeros), Glorot classifier.

    ``students`` (global indices) draws only that shard of the group — each student has its own
    labelled stream, so a shard is bit-identical to the same rows of the full group."""
    H, F, V, P, NL = cfg.hidden, cfg.ffn, cfg.vocab, cfg.max_pos, cfg.n_layers
    index = list(range(n_students)) if students is None else [int(i) for i in students]
    if any(not 0 <= i < n_students for i in index):
        raise ValueError("student index out of range")
    K = len(index)
    std = 0.02
    word = np.empty((K, V, H), np.float16)
    pos = np.empty((K, P, H), np.float16)
    typ = np.empty((K, H), np.float16)
    eg = np.empty((K, H), np.float32)
    eb = np.empty((K, H), np.float32)
    wq = np.empty((NL, K, 3 * H, H), np.float16)
    bq = np.empty((NL, K, 3 * H), np.float32)
    wo = np.empty((NL, K, H, H), np.float16)
    bo = np.empty((NL, K, H), np.float32)
    g1 = np.empty((NL, K, H), np.float32)
    be1 = np.empty((NL, K, H), np.float32)
    w1 = np.empty((NL, K, F, H), np.float16)
    b1 = np.empty((NL, K, F), np.float32)
    w2 = np.empty((NL, K, H, F), np.float16)
    b2 = np.empty((NL, K, H), np.float32)
    g2 = np.empty((NL, K, H), np.float32)
    be2 = np.empty((NL, K, H), np.float32)
    wp = np.empty((K, H, H), np.float16)
    bp = np.empty((K, H), np.float32)

    def nrm(rng, shape, s):
        return rng.standard_normal(size=shape, dtype=np.float32) * np.float32(s)

    for m, gidx in enumerate(index):
        rng = rng_for(seed, f"bert-student-{gidx}")
        word[m] = nrm(rng, (V, H), std)
        pos[m] = nrm(rng, (P, H), std)
        typ[m] = nrm(rng, (H,), std)
        eg[m] = 1.0 + nrm(rng, (H,), 0.1)
        eb[m] = nrm(rng, (H,), 0.05)
        for l in range(NL):
            wq[l, m] = nrm(rng, (3 * H, H), std)
            bq[l, m] = nrm(rng, (3 * H,), std)
            wo[l, m] = nrm(rng, (H, H), std)
            bo[l, m] = nrm(rng, (H,), std)
            g1[l, m] = 1.0 + nrm(rng, (H,), 0.1)
            be1[l, m] = nrm(rng, (H,), 0.05)
            w1[l, m] = nrm(rng, (F, H), std)
            b1[l, m] = nrm(rng, (F,), std)
            w2[l, m] = nrm(rng, (H, F), std)
            b2[l, m] = nrm(rng, (H,), std)
            g2[l, m] = 1.0 + nrm(rng, (H,), 0.1)
            be2[l, m] = nrm(rng, (H,), 0.05)
        wp[m] = nrm(rng, (H, H), std)
        bp[m] = nrm(rng, (H,), std)
    crng = rng_for(seed, "classifier")
    limit = math.sqrt(6.0 / (H + cfg.n_classes))  # DenseLayer.init -> _glorot_uniform (nnkernel.py:24-26, :55-56)
    w_cls = _f32(crng.uniform(-limit, limit, size=(cfg.n_classes, H)))
    b_cls = _f32(crng.normal(0.0, 0.02, size=cfg.n_classes))
    alpha = _alpha_draw(seed, n_students)[index]
    return BertGroupWeights(cfg, word, pos, typ, eg, eb, wq, bq, wo, bo, g1, be1, w1, b1, w2, b2, g2, be2, wp, bp,
                            alpha, w_cls, b_cls)


# --------------------------------------------------------------------------- dense kind
def _pad_to(n: int, m: int) -> int:
    return ((n + m - 1) // m) * m


@dataclass
class DenseGroupWeights:
    """Reference ``StudentModel`` group (nnkernel.py:256-301), fp16/fp32-rounded and zero-padded.

    Padding is exact: padded output features get zero weights and zero bias (tanh(0) = 0), and
    padded input features meet zero weight columns, so the logical result is unchanged.
    """

    d_in: int
    rep_dim: int
    depth: int
    n_classes: int
    w_in: np.ndarray      # f16 [K, Hp, Dp]
    b_in: np.ndarray      # f32 [K, Hp]
    w_layers: np.ndarray  # f16 [depth, K, Hp, Hp]
    b_layers: np.ndarray  # f32 [depth, K, Hp]
    alpha: np.ndarray     # f32 [K]
    w_cls: np.ndarray     # f32 [C, Hp]
    b_cls: np.ndarray     # f32 [C]
    # fp16 lo terms W - fp16(W) of float64 source weights (None: the fp16 weights are exact). The
    # engine then multiplies (W_hi + W_lo)(x_hi + x_lo) - W_lo x_lo: ~22-bit operands, so a
    # reference-trained float64 checkpoint reproduces the reference's own logits (ABI v3).
    w_in_lo: np.ndarray | None = None      # f16 [K, Hp, Dp]
    w_layers_lo: np.ndarray | None = None  # f16 [depth, K, Hp, Hp]
    kind: str = field(default="dense", init=False)

    @property
    def n_students(self) -> int:
        return int(self.alpha.shape[0])

    @property
    def hidden_padded(self) -> int:
        return int(self.w_in.shape[1])

    @property
    def d_in_padded(self) -> int:
        return int(self.w_in.shape[2])

    @property
    def exact_weights(self) -> bool:
        """True when the lo terms are carried (the engine runs the 3-product hi/lo projections)."""
        return self.w_in_lo is not None

    def subset(self, idx) -> "DenseGroupWeights":
        idx = np.asarray(idx, dtype=np.int64)
        lo = {}
        if self.exact_weights:
            lo = dict(w_in_lo=np.ascontiguousarray(self.w_in_lo[idx]),
                      w_layers_lo=np.ascontiguousarray(self.w_layers_lo[:, idx]))
        return replace(self, w_in=np.ascontiguousarray(self.w_in[idx]), b_in=np.ascontiguousarray(self.b_in[idx]),
                       w_layers=np.ascontiguousarray(self.w_layers[:, idx]),
                       b_layers=np.ascontiguousarray(self.b_layers[:, idx]),
                       alpha=np.ascontiguousarray(self.alpha[idx]), **lo)

    # Unpadded per-student arrays in float64 exactly as the engine represents them (hi + lo when
    # the lo terms are carried) — what the oracle is fed for "identical weights" parity.
    def student_layers(self, m: int) -> list[tuple[np.ndarray, np.ndarray]]:
        H, D = self.rep_dim, self.d_in

        def mat(hi, lo):
            v = hi.astype(np.float64)
            return v if lo is None else v + lo.astype(np.float64)

        out = [(mat(self.w_in[m, :H, :D], None if self.w_in_lo is None else self.w_in_lo[m, :H, :D]),
                self.b_in[m, :H].astype(np.float64))]
        for l in range(self.depth):
            lo = None if self.w_layers_lo is None else self.w_layers_lo[l, m, :H, :H]
            out.append((mat(self.w_layers[l, m, :H, :H], lo), self.b_layers[l, m, :H].astype(np.float64)))
        return out

    def classifier(self) -> tuple[np.ndarray, np.ndarray]:
        return self.w_cls[:, : self.rep_dim].astype(np.float64), self.b_cls.astype(np.float64)


def dense_group_from_arrays(students: list[list[tuple[np.ndarray, np.ndarray]]], multipliers, classifier,
                            exact: bool = True) -> DenseGroupWeights:
    """Build from per-student [(W_in, b_in), (W_1, b_1), ...] lists and classifier (W_c, b_c).

    exact: keep the fp16 lo terms of weights that fp16 does not represent (float64 sources such as
    the reference's trained checkpoints); with exact=False, or when every weight is already an fp16
    value, the group carries fp16 weights only (one weight operand per projection)."""
    K = len(students)
    if K == 0:
        raise ValueError("empty ensemble")
    if len(multipliers) != K:
        raise ValueError("students and multipliers must have equal length")  # distill.py:150-151
    if float(multipliers[0]) != 1.0:
        raise ValueError("the first multiplier must be exactly 1")  # distill.py:152-153
    if classifier is None:
        raise ValueError("ensemble has no trained classifier")  # distill.py:510-511
    w0 = np.asarray(students[0][0][0])
    rep_dim, d_in = w0.shape
    depth = len(students[0]) - 1
    if depth < 2:
        raise ValueError("student needs at least 2 layers")  # nnkernel.py:265-266
    Hp, Dp = _pad_to(rep_dim, 128), _pad_to(d_in, 64)
    w_in = np.zeros((K, Hp, Dp), np.float16)
    b_in = np.zeros((K, Hp), np.float32)
    w_l = np.zeros((depth, K, Hp, Hp), np.float16)
    b_l = np.zeros((depth, K, Hp), np.float32)
    for m, layers in enumerate(students):
        if len(layers) != depth + 1:
            raise ValueError("all students must have the same depth")
        W, b = layers[0]
        if np.asarray(W).shape != (rep_dim, d_in):
            raise ValueError("all students must share d_in and rep_dim")
        w_in[m, :rep_dim, :d_in] = np.asarray(W, dtype=np.float64)
        b_in[m, :rep_dim] = np.asarray(b, dtype=np.float64)
        for l, (W, b) in enumerate(layers[1:]):
            if np.asarray(W).shape != (rep_dim, rep_dim):
                raise ValueError("hidden layers must be rep_dim x rep_dim")
            w_l[l, m, :rep_dim, :rep_dim] = np.asarray(W, dtype=np.float64)
            b_l[l, m, :rep_dim] = np.asarray(b, dtype=np.float64)
    Wc, bc = classifier
    Wc = np.asarray(Wc, dtype=np.float64)
    if Wc.shape[1] != rep_dim:
        raise ValueError(f"classifier in_dim {Wc.shape[1]} does not match rep_dim {rep_dim}")
    w_cls = np.zeros((Wc.shape[0], Hp), np.float32)
    w_cls[:, :rep_dim] = Wc
    lo = {}
    if exact:
        w_in_lo = np.zeros_like(w_in)
        w_l_lo = np.zeros_like(w_l)
        for m, layers in enumerate(students):
            W = np.asarray(layers[0][0], dtype=np.float64)
            w_in_lo[m, :rep_dim, :d_in] = W - w_in[m, :rep_dim, :d_in].astype(np.float64)
            for l, (W, _) in enumerate(layers[1:]):
                W = np.asarray(W, dtype=np.float64)
                w_l_lo[l, m, :rep_dim, :rep_dim] = W - w_l[l, m, :rep_dim, :rep_dim].astype(np.float64)
        if w_in_lo.any() or w_l_lo.any():
            lo = dict(w_in_lo=w_in_lo, w_layers_lo=w_l_lo)
    return DenseGroupWeights(d_in, rep_dim, depth, int(Wc.shape[0]), w_in, b_in, w_l, b_l,
                             _f32(np.asarray(multipliers, dtype=np.float64)), w_cls, _f32(bc), **lo)


def dense_group_from_ensemble(state) -> DenseGroupWeights:
    """Snapshot a reference ``EnsembleState`` (distill.py:139-178) — duck-typed, no import needed."""
    students = []
    for s in state.students:
        layers = [(s.input_proj.weight, s.input_proj.bias)] + [(l.weight, l.bias) for l in s.layers]
        for lay in [s.input_proj, *s.layers]:
            if lay.activation != "tanh":
                raise ValueError("the engine's dense student applies tanh on every layer (nnkernel.py:272-273)")
        students.append(layers)
    clf = state.classifier
    if clf is not None and getattr(clf, "activation", "identity") != "identity":
        raise ValueError("classifier must be an identity DenseLayer (distill.py:535)")
    return dense_group_from_arrays(students, list(state.multipliers),
                                   None if clf is None else (clf.weight, clf.bias))


def random_dense_group(d_in: int, rep_dim: int, depth: int, n_students: int, n_classes: int = 2,
                       seed: int = 0, exact: bool = True) -> DenseGroupWeights:
    """Glorot-uniform students as ``StudentModel.build`` draws them (nnkernel.py:24-26, :270-274),
    with small random biases so the bias path is exercised."""
    students = []
    for m in range(n_students):
        rng = rng_for(seed, f"dense-student-{m}")
        layers = []
        dims = [(rep_dim, d_in)] + [(rep_dim, rep_dim)] * depth
        for out_dim, in_dim in dims:
            limit = math.sqrt(6.0 / (in_dim + out_dim))
            layers.append((rng.uniform(-limit, limit, size=(out_dim, in_dim)), rng.normal(0, 0.05, size=out_dim)))
        students.append(layers)
    crng = rng_for(seed, "classifier")
    limit = math.sqrt(6.0 / (rep_dim + n_classes))
    clf = (crng.uniform(-limit, limit, size=(n_classes, rep_dim)), crng.normal(0, 0.05, size=n_classes))
    return dense_group_from_arrays(students, [float(a) for a in _alpha_draw(seed, n_students)], clf, exact=exact)

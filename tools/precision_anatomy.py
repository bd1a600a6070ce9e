"""Which fp16 rounding of the engine's activations moves the logits? (CPU, float64 oracle with
round-to-fp16 inserted at one point at a time; no GPU.) Points: the GEMM inputs after each LayerNorm
('ln'; 'cls' = only the CLS row the pooler reads; 'lnmid' = all but that row), the stored QKV ('qkv'), the attention probabilities ('p'), the attention context ('ctx'), the
GELU output ('gelu'). Prints the logit error relative to max|logit| of the exact oracle.

    python tools/precision_anatomy.py
"""
import sys

import numpy as np

sys.path.insert(0, ".")
import oracle.bert as ob  # noqa: E402
from oracle.dense import IDENTITY, TANH, dense_layer, ensemble_rep  # noqa: E402
from paper_2408_12526_b200 import PRESETS, random_bert_group  # noqa: E402


def h(x, on):
    return x.astype(np.float16).astype(np.float64) if on else x


def encode(o, m, ids, pts):
    cfg, s = o.cfg, o.student(m)
    L = len(ids)
    x = s["word"][ids].astype(np.float64) + s["pos"][:L].astype(np.float64) + s["type"]
    x = ob.layer_norm(x, *s["emb_ln"], cfg.ln_eps)
    nh, hd, H = cfg.n_heads, cfg.head_dim, cfg.hidden
    for lay in s["layers"]:
        qkv = h(dense_layer(*lay["qkv"], h(x, "ln" in pts or "lnmid" in pts), IDENTITY), "qkv" in pts)
        q, k, v = (qkv[:, i * H:(i + 1) * H].reshape(L, nh, hd) for i in range(3))
        sc = np.einsum("qhd,khd->hqk", q, k) / np.sqrt(hd)
        p = np.exp(sc - sc.max(-1, keepdims=True))
        p = h(p, "p" in pts) / p.sum(-1, keepdims=True)  # unnormalised P is the MMA operand
        ctx = h(np.einsum("hqk,khd->qhd", p, v).reshape(L, H), "ctx" in pts)
        x = ob.layer_norm(x + dense_layer(*lay["o"], ctx, IDENTITY), *lay["ln1"], cfg.ln_eps)
        f = h(ob.gelu(dense_layer(*lay["ffn1"], h(x, "ln" in pts or "lnmid" in pts), IDENTITY)), "gelu" in pts)
        x = ob.layer_norm(x + dense_layer(*lay["ffn2"], f, IDENTITY), *lay["ln2"], cfg.ln_eps)
    return x


def logits(o, ids, pts):
    finals = []
    for m in range(o.n_students):
        cls = h(encode(o, m, ids, pts)[:1], "ln" in pts or "cls" in pts)
        finals.append(dense_layer(*o.student(m)["pool"], cls, TANH))
    return dense_layer(o.w_cls, o.b_cls, ensemble_rep(finals, o.alpha, o.n_students), IDENTITY)[0]


for name, seed, L in (("large", 31, 384), ("base", 31, 512), ("large", 32, 512)):
    cfg, _ = PRESETS[name]
    o = ob.OracleBertGroup(random_bert_group(cfg, 2, seed=seed))
    ids = np.r_[101, np.random.default_rng(L + seed).integers(1000, 30522, size=L - 1)].astype(np.int64)
    z0 = logits(o, ids, set())
    for pts in (["ln"], ["cls"], ["qkv"], ["p"], ["ctx"], ["gelu"], ["ln", "qkv", "p", "ctx", "gelu"],
                ["qkv", "p", "ctx", "gelu", "lnmid"]):
        z = logits(o, ids, set(pts))
        print(f"{name} seed {seed} L={L} fp16 at {'+'.join(pts):20s} logits rel {np.abs(z - z0).max() / np.abs(z0).max():.2e}",
              flush=True)

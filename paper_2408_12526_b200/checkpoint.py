"""The reference's JSON checkpoints <-> engine weights.

Schemas (restated, not imported): ``dense-model-checkpoint-v1`` (nnkernel.py:471-558) and
``ensemble-checkpoint-v1`` (distill.py:586-612). In "binary" mode arrays are base64 little-endian
float64 (bit exact, nnkernel.py:474-477); in "json" mode decimal lists. Non-finite values are
rejected (nnkernel.py:486-487), as are unknown schemas/kinds (nnkernel.py:535-536, :547).

BERT-student extension (the paper's students, which the artifact cannot express): a student entry
of an ensemble-checkpoint-v1 container with ``"kind": "bert-student"`` inside the same
dense-model-checkpoint-v1 schema. Every affine map is the reference's layer dict
(``_layer_to_dict``, nnkernel.py:490-497: out_dim, in_dim, activation, weight, bias) — QKV and O
with identity, FFN1 with "gelu" (erf), FFN2 identity, the pooler with tanh; embeddings and
LayerNorm vectors are {"shape", "data"} arrays in the same float64 encoding; "config" carries the
architecture. The group container (multipliers, identity classifier) is unchanged
(distill.py:586-595), so a group saves and loads with a bit-exact round trip.
"""
from __future__ import annotations

import base64
import json

import numpy as np

from .weights import BertConfig, BertGroupWeights, DenseGroupWeights, dense_group_from_arrays

MODEL_SCHEMA = "dense-model-checkpoint-v1"
ENSEMBLE_SCHEMA = "ensemble-checkpoint-v1"
BERT_KIND = "bert-student"


def _encode_array(arr: np.ndarray, mode: str):
    """nnkernel.py:474-477: base64 little-endian float64 ("binary") or a decimal list ("json")."""
    a = np.asarray(arr, dtype=np.float64)
    if mode == "binary":
        return base64.b64encode(a.astype("<f8").tobytes()).decode("ascii")
    if mode == "json":
        return a.ravel().tolist()
    raise ValueError(f"unknown checkpoint mode {mode!r}")


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
    if any(s.get("kind") == BERT_KIND for s in d["students"]):
        raise ValueError("BERT-student ensemble: use bert_group_from_dict")
    students = [_student_layers(s) for s in d["students"]]
    clf = None
    if d["classifier"] is not None:
        w, b, act = _layer(d["classifier"], d["mode"])
        if act != "identity":
            raise ValueError("classifier must be an identity layer (distill.py:535)")
        clf = (w, b)
    return students, list(d["multipliers"]), clf


# --------------------------------------------------------------------------- BERT-student kind
def _layer_dict(w, b, activation: str, mode: str) -> dict:
    """The reference's layer dict (nnkernel.py:490-497)."""
    w = np.asarray(w, dtype=np.float64)
    return {"out_dim": int(w.shape[0]), "in_dim": int(w.shape[1]), "activation": activation,
            "weight": _encode_array(w, mode), "bias": _encode_array(b, mode)}


def _array_dict(a, mode: str) -> dict:
    a = np.asarray(a)
    return {"shape": list(a.shape), "data": _encode_array(a, mode)}


def _array(d: dict, mode: str) -> np.ndarray:
    return _decode_array(d["data"], tuple(d["shape"]), mode)


def bert_student_to_dict(w: BertGroupWeights, m: int, mode: str = "binary") -> dict:
    """Student m of a BERT-kind group as a dense-model-checkpoint-v1 dict of kind "bert-student"."""
    c = w.cfg
    H = c.hidden
    layers = []
    for l in range(c.n_layers):
        layers.append({
            "qkv": _layer_dict(w.w_qkv[l, m], w.b_qkv[l, m], "identity", mode),
            "o": _layer_dict(w.w_o[l, m], w.b_o[l, m], "identity", mode),
            "ln1_gamma": _array_dict(w.ln1_gamma[l, m], mode), "ln1_beta": _array_dict(w.ln1_beta[l, m], mode),
            "ffn1": _layer_dict(w.w_ffn1[l, m], w.b_ffn1[l, m], "gelu", mode),
            "ffn2": _layer_dict(w.w_ffn2[l, m], w.b_ffn2[l, m], "identity", mode),
            "ln2_gamma": _array_dict(w.ln2_gamma[l, m], mode), "ln2_beta": _array_dict(w.ln2_beta[l, m], mode),
        })
    assert w.w_qkv.shape[2] == 3 * H
    return {
        "schema": MODEL_SCHEMA, "mode": mode, "kind": BERT_KIND,
        "config": {"hidden": c.hidden, "n_layers": c.n_layers, "n_heads": c.n_heads, "ffn": c.ffn,
                   "vocab": c.vocab, "max_pos": c.max_pos, "ln_eps": c.ln_eps},
        "embeddings": {"word": _array_dict(w.word_emb[m], mode), "position": _array_dict(w.pos_emb[m], mode),
                       "token_type": _array_dict(w.type_emb[m], mode),
                       "ln_gamma": _array_dict(w.emb_ln_gamma[m], mode),
                       "ln_beta": _array_dict(w.emb_ln_beta[m], mode)},
        "layers": layers,
        "pooler": _layer_dict(w.w_pool[m], w.b_pool[m], "tanh", mode),
    }


def bert_group_to_dict(w: BertGroupWeights, mode: str = "binary") -> dict:
    """A BERT-kind group as an ensemble-checkpoint-v1 dict (distill.py:586-595)."""
    return {
        "schema": ENSEMBLE_SCHEMA, "mode": mode,
        "multipliers": [float(a) for a in w.alpha],
        "students": [bert_student_to_dict(w, m, mode) for m in range(w.n_students)],
        "classifier": _layer_dict(w.w_cls, w.b_cls, "identity", mode),
    }


def _check_layer(d: dict, shape: tuple[int, int], activation: str, mode: str):
    if (d["out_dim"], d["in_dim"]) != shape:
        raise ValueError(f"layer shape {(d['out_dim'], d['in_dim'])} != {shape}")
    if d["activation"] != activation:
        raise ValueError(f"layer activation {d['activation']!r} != {activation!r}")
    w, b, _ = _layer(d, mode)
    return w, b


def bert_group_from_dict(d: dict) -> BertGroupWeights:
    """ensemble-checkpoint-v1 with bert-student entries -> engine weights (matrices rounded to fp16,
    vectors to fp32: exact for weights the engine saved)."""
    if d.get("schema") != ENSEMBLE_SCHEMA:
        raise ValueError("not an ensemble checkpoint")
    mode = d["mode"]
    studs = d["students"]
    if not studs:
        raise ValueError("ensemble has no students")
    for s in studs:
        if s.get("schema") != MODEL_SCHEMA or s.get("kind") != BERT_KIND:
            raise ValueError("every student must be a bert-student dense-model-checkpoint-v1 entry")
    cfg = BertConfig(**studs[0]["config"])
    if any(BertConfig(**s["config"]) != cfg for s in studs):
        raise ValueError("students of one group must share an architecture")
    mult = [float(a) for a in d["multipliers"]]
    if len(mult) != len(studs) or mult[0] != 1.0:
        raise ValueError("one multiplier per student, the first equal to 1 (distill.py:152-153)")
    if d["classifier"] is None:
        raise ValueError("the group needs a classifier (distill.py:510-511)")
    H, F, NL, K = cfg.hidden, cfg.ffn, cfg.n_layers, len(studs)
    f16 = lambda a: np.ascontiguousarray(np.stack(a), dtype=np.float16)  # noqa: E731
    f32 = lambda a: np.ascontiguousarray(np.stack(a), dtype=np.float32)  # noqa: E731
    per = {n: [] for n in ["word", "pos", "type", "eg", "eb", "wp", "bp"]}
    lay = {n: [[] for _ in range(NL)] for n in ["wq", "bq", "wo", "bo", "g1", "b1", "w1", "c1", "w2", "c2", "g2", "b2"]}
    for s in studs:
        e = s["embeddings"]
        per["word"].append(_array(e["word"], mode))
        per["pos"].append(_array(e["position"], mode))
        per["type"].append(_array(e["token_type"], mode))
        per["eg"].append(_array(e["ln_gamma"], mode))
        per["eb"].append(_array(e["ln_beta"], mode))
        if len(s["layers"]) != NL:
            raise ValueError("layer count does not match the config")
        for l, ld in enumerate(s["layers"]):
            wq, bq = _check_layer(ld["qkv"], (3 * H, H), "identity", mode)
            wo, bo = _check_layer(ld["o"], (H, H), "identity", mode)
            w1, c1 = _check_layer(ld["ffn1"], (F, H), "gelu", mode)
            w2, c2 = _check_layer(ld["ffn2"], (H, F), "identity", mode)
            for n, v in (("wq", wq), ("bq", bq), ("wo", wo), ("bo", bo), ("w1", w1), ("c1", c1), ("w2", w2),
                         ("c2", c2), ("g1", _array(ld["ln1_gamma"], mode)), ("b1", _array(ld["ln1_beta"], mode)),
                         ("g2", _array(ld["ln2_gamma"], mode)), ("b2", _array(ld["ln2_beta"], mode))):
                lay[n][l].append(v)
        wp, bp = _check_layer(s["pooler"], (H, H), "tanh", mode)
        per["wp"].append(wp)
        per["bp"].append(bp)
    wc, bc, act = _layer(d["classifier"], mode)
    if act != "identity" or wc.shape[1] != H:
        raise ValueError("classifier must be an identity layer over the students' width (distill.py:535)")
    L = lambda n, conv: np.ascontiguousarray(np.stack([conv(lay[n][l]) for l in range(NL)]))  # noqa: E731
    cfg = BertConfig(hidden=H, n_layers=NL, n_heads=cfg.n_heads, ffn=F, vocab=cfg.vocab, max_pos=cfg.max_pos,
                     n_classes=int(wc.shape[0]), ln_eps=cfg.ln_eps)
    return BertGroupWeights(
        cfg, f16(per["word"]), f16(per["pos"]), f16(per["type"]), f32(per["eg"]), f32(per["eb"]),
        L("wq", f16), L("bq", f32), L("wo", f16), L("bo", f32), L("g1", f32), L("b1", f32), L("w1", f16),
        L("c1", f32), L("w2", f16), L("c2", f32), L("g2", f32), L("b2", f32), f16(per["wp"]), f32(per["bp"]),
        np.asarray(mult, np.float32), np.ascontiguousarray(wc, np.float32), np.ascontiguousarray(bc, np.float32))


def save_bert_ensemble(w: BertGroupWeights, path, mode: str = "binary") -> None:
    """save_ensemble (distill.py:604-607) for a BERT-kind group."""
    with open(path, "w", encoding="utf-8") as fh:
        json.dump(bert_group_to_dict(w, mode), fh, indent=1)
        fh.write("\n")


def load_ensemble_weights(path) -> DenseGroupWeights | BertGroupWeights:
    """load_ensemble (distill.py:610-612) -> engine weights, dense or BERT-student kind."""
    with open(path, "r", encoding="utf-8") as fh:
        d = json.load(fh)
    if d.get("schema") == ENSEMBLE_SCHEMA and any(s.get("kind") == BERT_KIND for s in d.get("students", [])):
        return bert_group_from_dict(d)
    return dense_group_from_arrays(*ensemble_arrays_from_dict(d))

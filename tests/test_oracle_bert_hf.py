"""External pin of the BERT-student oracle (SURVEY §8c "parity unpinned"): oracle/bert.py against a
published BERT implementation, transformers' ``BertModel``, in float64 on the same weights.

The reference artifact has no transformer code; the paper defines the student as a
residual post-LN BERT encoder initialised from BERT whose output
is the pooled final representation, summed over students. HF
``BertModel`` with ``hidden_act="gelu"`` (erf GELU), LayerNorm eps 1e-12, token type 0 and absolute
positions restarting at 0 per sequence is exactly that student; its ``pooler_output`` is
tanh(W_p h_CLS + b_p). Every student of a group, and the group logits built from the pooled
outputs with the reference's boosting sum (distill.py:169-178) + classifier, must match the
oracle to float64 rounding.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
transformers = pytest.importorskip("transformers")


def _hf_student(w, m):
    """A float64 transformers.BertModel holding student m of a BertGroupWeights."""
    cfg = w.cfg
    hf_cfg = transformers.BertConfig(
        vocab_size=cfg.vocab, hidden_size=cfg.hidden, num_hidden_layers=cfg.n_layers,
        num_attention_heads=cfg.n_heads, intermediate_size=cfg.ffn, hidden_act="gelu",
        max_position_embeddings=cfg.max_pos, type_vocab_size=2, layer_norm_eps=cfg.ln_eps,
        hidden_dropout_prob=0.0, attention_probs_dropout_prob=0.0, attn_implementation="eager")
    model = transformers.BertModel(hf_cfg, add_pooling_layer=True).double().eval()
    H = cfg.hidden
    t = lambda a: torch.from_numpy(np.asarray(a, dtype=np.float64).copy())  # noqa: E731
    with torch.no_grad():
        emb = model.embeddings
        emb.word_embeddings.weight.copy_(t(w.word_emb[m]))
        emb.position_embeddings.weight.copy_(t(w.pos_emb[m]))
        emb.token_type_embeddings.weight.zero_()
        emb.token_type_embeddings.weight[0].copy_(t(w.type_emb[m]))
        emb.LayerNorm.weight.copy_(t(w.emb_ln_gamma[m]))
        emb.LayerNorm.bias.copy_(t(w.emb_ln_beta[m]))
        for l, layer in enumerate(model.encoder.layer):
            wq, bq = w.w_qkv[l, m], w.b_qkv[l, m]
            att = layer.attention
            for i, lin in enumerate((att.self.query, att.self.key, att.self.value)):
                lin.weight.copy_(t(wq[i * H:(i + 1) * H]))
                lin.bias.copy_(t(bq[i * H:(i + 1) * H]))
            att.output.dense.weight.copy_(t(w.w_o[l, m]))
            att.output.dense.bias.copy_(t(w.b_o[l, m]))
            att.output.LayerNorm.weight.copy_(t(w.ln1_gamma[l, m]))
            att.output.LayerNorm.bias.copy_(t(w.ln1_beta[l, m]))
            layer.intermediate.dense.weight.copy_(t(w.w_ffn1[l, m]))
            layer.intermediate.dense.bias.copy_(t(w.b_ffn1[l, m]))
            layer.output.dense.weight.copy_(t(w.w_ffn2[l, m]))
            layer.output.dense.bias.copy_(t(w.b_ffn2[l, m]))
            layer.output.LayerNorm.weight.copy_(t(w.ln2_gamma[l, m]))
            layer.output.LayerNorm.bias.copy_(t(w.ln2_beta[l, m]))
        model.pooler.dense.weight.copy_(t(w.w_pool[m]))
        model.pooler.dense.bias.copy_(t(w.b_pool[m]))
    return model


def _hf_pooled(model, ids):
    with torch.no_grad():
        x = torch.from_numpy(np.asarray(ids, np.int64))[None, :]
        out = model(input_ids=x, token_type_ids=torch.zeros_like(x), attention_mask=torch.ones_like(x))
    return out.pooler_output[0].numpy(), out.last_hidden_state[0].numpy()


@pytest.mark.parametrize("hidden,heads,layers", [(128, 4, 2), (256, 4, 1)])
def test_oracle_student_matches_transformers_bert(hidden, heads, layers):
    from oracle.bert import OracleBertGroup
    from paper_2408_12526_b200 import BertConfig, random_bert_group

    cfg = BertConfig(hidden=hidden, n_heads=heads, n_layers=layers, vocab=1200, max_pos=80)
    w = random_bert_group(cfg, 2, seed=hidden + layers)
    orc = OracleBertGroup(w)
    rng = np.random.default_rng(hidden)
    for m in range(2):
        model = _hf_student(w, m)
        for L in (1, 7, 50, 80):
            ids = np.r_[101, rng.integers(200, cfg.vocab, size=L - 1)].astype(np.int64)
            pooled_hf, hidden_hf = _hf_pooled(model, ids)
            hidden_or = orc.encode(m, ids)
            pooled_or = orc.pooled(m, [ids])[0]
            assert np.abs(hidden_or - hidden_hf).max() <= 1e-12
            assert np.abs(pooled_or - pooled_hf).max() <= 1e-12


def test_oracle_group_logits_from_transformers_pooled_outputs():
    """The group head on HF pooled outputs (boosting sum in student order + classifier, bias once)
    equals the oracle's logits for every prefix k (packed ragged batch, positions restart per sequence)."""
    from oracle.bert import OracleBertGroup
    from oracle.dense import IDENTITY, dense_layer, ensemble_rep
    from paper_2408_12526_b200 import BertConfig, random_bert_group

    cfg = BertConfig(hidden=128, n_heads=4, n_layers=2, vocab=1200, max_pos=64)
    K = 3
    w = random_bert_group(cfg, K, seed=9)
    orc = OracleBertGroup(w)
    rng = np.random.default_rng(9)
    seqs = [np.r_[101, rng.integers(200, cfg.vocab, size=L - 1)].astype(np.int64) for L in (5, 64, 17)]
    pooled = [np.stack([_hf_pooled(_hf_student(w, m), s)[0] for s in seqs]) for m in range(K)]
    for k in range(1, K + 1):
        rep_hf = ensemble_rep(pooled, [float(a) for a in w.alpha], k)
        z_hf = dense_layer(w.w_cls.astype(np.float64), w.b_cls.astype(np.float64), rep_hf, IDENTITY)
        ids = np.concatenate(seqs)
        cu = np.r_[0, np.cumsum([len(s) for s in seqs])]
        rep_or, z_or = orc.forward_packed(ids, cu, k)
        assert np.abs(rep_or - rep_hf).max() <= 1e-12
        assert np.abs(z_or - z_hf).max() <= 1e-12

"""Worst prefix-k case of the r2 sweep: engine error vs the float64 oracle with the engine's remaining
fp16 rounding points emulated (QKV outputs of both layers, P of the layer-1 attention), per attention
kernel. python tools/diag_prefix.py [config seed L k]"""
import os, subprocess, sys
import numpy as np
sys.path.insert(0, ".")

def emulate(name, K, seed, L, k, pts):
    import oracle.bert as ob
    from oracle.dense import IDENTITY, TANH, dense_layer, ensemble_rep
    from paper_2408_12526_b200 import PRESETS, random_bert_group
    cfg, _ = PRESETS[name]
    o = ob.OracleBertGroup(random_bert_group(cfg, K, seed=seed, students=range(k)))
    rng = np.random.default_rng(seed)
    reqs = [np.r_[101, rng.integers(1000, cfg.vocab, size=Lx - 1)].astype(np.int64) for Lx in (16, 128, 384, 512)]
    ids = reqs[[16, 128, 384, 512].index(L)]
    h = lambda x, on: x.astype(np.float16).astype(np.float64) if on else x
    def enc(m):
        s = o.student(m); cfg = o.cfg
        x = s["word"][ids].astype(np.float64) + s["pos"][:L].astype(np.float64) + s["type"]
        x = ob.layer_norm(x, *s["emb_ln"], cfg.ln_eps)
        nh, hd, H = cfg.n_heads, cfg.head_dim, cfg.hidden
        nl = len(s["layers"])
        for li, lay in enumerate(s["layers"]):
            last = li == nl - 1
            qkv = h(dense_layer(*lay["qkv"], x, IDENTITY),
                    "qkv" in pts or (f"qkv{li}" in pts) or ("qkvL" in pts and last))
            if li == 0:  # per-operand rounding of the first layer's attention inputs
                for nm, i in (("q0", 0), ("k0", 1), ("v0", 2)):
                    if nm in pts:
                        qkv[:, i * H:(i + 1) * H] = h(qkv[:, i * H:(i + 1) * H], True)
            q, kk, v = (qkv[:, i * H:(i + 1) * H].reshape(L, nh, hd) for i in range(3))
            sc = np.einsum("qhd,khd->hqk", q, kk) / np.sqrt(hd)
            p = np.exp(sc - sc.max(-1, keepdims=True))
            p = h(p, "p" in pts and not last) / p.sum(-1, keepdims=True)
            ctx = np.einsum("hqk,khd->qhd", p, v).reshape(L, H)
            x = ob.layer_norm(x + dense_layer(*lay["o"], ctx, IDENTITY), *lay["ln1"], cfg.ln_eps)
            f = ob.gelu(dense_layer(*lay["ffn1"], x, IDENTITY))
            x = ob.layer_norm(x + dense_layer(*lay["ffn2"], f, IDENTITY), *lay["ln2"], cfg.ln_eps)
        return x
    fin = [dense_layer(*o.student(m)["pool"], enc(m)[:1], TANH) for m in range(k)]
    return dense_layer(o.w_cls, o.b_cls, ensemble_rep(fin, o.alpha, k), IDENTITY)[0], ids

name, seed, L, k = (sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])) if len(sys.argv) > 4 else ("k32", 106, 16, 9)
from paper_2408_12526_b200 import PRESETS
K = PRESETS[name][1]
z0, ids = emulate(name, K, seed, L, k, set())
for pts in (["qkv0"], ["q0"], ["k0"], ["v0"], ["p"], ["q0", "k0"], ["q0", "k0", "p"], ["v0", "p"]):
    z, _ = emulate(name, K, seed, L, k, set(pts))
    print(f"emulated fp16 at {'+'.join(pts):8s}: {np.abs(z - z0).max() / np.abs(z0).max():.2e}  (max|z| {np.abs(z0).max():.4f})")
if os.environ.get("DIAG_CHILD") is None:
    np.save("/tmp/diag_ref.npy", z0)
    for kind in ("", "0", "1", "2", "3"):
        env = dict(os.environ, DIAG_CHILD="1")
        if kind:
            env["SP_ATTN_TC"] = kind
        code = (f"import sys,numpy as np; sys.path.insert(0,'.');"
                f"from paper_2408_12526_b200 import PRESETS, StudentGroup, random_bert_group;"
                f"cfg,K=PRESETS['{name}']; w=random_bert_group(cfg,K,seed={seed}); g=StudentGroup(w,max_tokens=512,max_seqs=1);"
                f"rng=np.random.default_rng({seed}); reqs=[np.r_[101, rng.integers(1000, cfg.vocab, size=Lx-1)].astype(np.int32) for Lx in (16,128,384,512)];"
                f"ids=reqs[[16,128,384,512].index({L})]; z=g.logits(ids,{k}); z0=np.load('/tmp/diag_ref.npy');"
                f"print('engine SP_ATTN_TC={kind or 'default'}:', '%.2e' % (np.abs(z-z0).max()/np.abs(z0).max()))")
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
        print(r.stdout.strip() or r.stderr[-400:])

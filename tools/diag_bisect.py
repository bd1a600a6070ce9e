import sys, numpy as np
sys.path.insert(0, ".")
from oracle.bert import OracleBertGroup
from oracle.dense import group_forward_weights
from paper_2408_12526_b200 import PRESETS, BertConfig, StudentGroup, random_bert_group, random_dense_group

def err(got, ref):
    got, ref = np.atleast_2d(got), np.atleast_2d(ref)
    return np.abs(got - ref).max() / np.abs(ref).max()

rng = np.random.default_rng(5)
def seqs(n, lo, hi):
    return [np.r_[101, rng.integers(1000, 30522, size=int(L) - 1)].astype(np.int32) for L in rng.integers(lo, hi + 1, size=n)]

def run(name, cfg, K, ss, **kw):
    w = random_bert_group(cfg, K, seed=3)
    g = StudentGroup(w, max_tokens=2048, max_seqs=64, **kw); o = OracleBertGroup(w)
    rep_ref, _ = o.forward(ss, 1)
    print(f"{name}: rep err k=1 {err(g.rep(ss, 1), rep_ref):.3e}", flush=True)

tiny = PRESETS["tiny"][0]
run("tiny 1seq L=40", tiny, 2, seqs(1, 40, 40))
run("tiny 1seq L=16", tiny, 2, seqs(1, 16, 16))
run("tiny 3seq", tiny, 2, seqs(3, 8, 64))
run("tiny 1 layer 1seq", BertConfig(hidden=128, n_heads=4, n_layers=1), 2, seqs(1, 40, 40))
run("tiny hd64 (2 heads) 1seq", BertConfig(hidden=128, n_heads=2), 2, seqs(1, 40, 40))
run("h256 hd64 1seq", BertConfig(hidden=256, n_heads=4), 2, seqs(1, 40, 40))
run("h256 hd32 1seq", BertConfig(hidden=256, n_heads=8), 2, seqs(1, 40, 40))
run("h768 1seq", BertConfig(hidden=768, n_heads=12), 2, seqs(1, 40, 40))
run("h768 3seq", BertConfig(hidden=768, n_heads=12), 2, seqs(3, 8, 64))
for (d, r) in [(8, 16), (64, 128), (128, 128), (768, 768), (64, 256)]:
    wd = random_dense_group(d, r, 2, 3, 2, 4)
    gd = StudentGroup(wd, max_tokens=512)
    x = np.random.default_rng(2).normal(size=(50, d))
    rep_ref, z_ref = group_forward_weights(wd, np.float16(x).astype(np.float64), 1)
    print(f"dense d={d} r={r}: rep err {err(gd.rep(x, 1), rep_ref):.3e}", flush=True)

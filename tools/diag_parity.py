"""Diagnostic: error anatomy of the engine vs the float64 oracle (prints, no asserts)."""
import sys, numpy as np
sys.path.insert(0, ".")
from oracle.bert import OracleBertGroup
from oracle.dense import group_forward_weights
from paper_2408_12526_b200 import PRESETS, StudentGroup, random_bert_group, random_dense_group

def stats(name, got, ref):
    got, ref = np.atleast_2d(got), np.atleast_2d(ref)
    d = np.abs(got - ref)
    rowmax = np.abs(ref).max(1)
    print(f"{name}: max|d|={d.max():.3e} global_rel={d.max()/np.abs(ref).max():.3e} "
          f"row_rel_max={(d.max(1)/rowmax).max():.3e} row_rel_med={np.median(d.max(1)/rowmax):.3e} "
          f"|ref| max={np.abs(ref).max():.3e} min_rowmax={rowmax.min():.3e}")

cfg, K = PRESETS["tiny"]
w = random_bert_group(cfg, K, seed=11)
g = StudentGroup(w, max_tokens=2048, max_seqs=64); o = OracleBertGroup(w)
rng = np.random.default_rng(101)
seqs = [np.r_[101, rng.integers(1000, 30522, size=int(L) - 1)].astype(np.int32) for L in rng.integers(8, 65, size=7)]
for k in (1, 4):
    rep_ref, z_ref = o.forward(seqs, k)
    stats(f"tiny k={k} rep", g.rep(seqs, k), rep_ref)
    stats(f"tiny k={k} logits", g.logits(seqs, k), z_ref)
# pooled of student 0 per element
print("pooled0 sample gpu", g.rep(seqs, 1)[0, :6]); print("pooled0 sample ref", o.forward(seqs, 1)[0][0, :6])
wd = random_dense_group(768, 768, 2, 8, 2, 8)
gd = StudentGroup(wd, max_tokens=256)
x = np.random.default_rng(3).normal(size=(256, 768))
rep_ref, z_ref = group_forward_weights(wd, np.float16(x).astype(np.float64))
stats("dense768 rep", gd.rep(x), rep_ref); stats("dense768 logits", gd.logits(x), z_ref)
cfg, K = PRESETS["base"]
wb = random_bert_group(cfg, K, seed=1); gb = StudentGroup(wb, max_tokens=1024, max_seqs=8); ob = OracleBertGroup(wb)
for L in (16, 100):
    ids = [np.r_[101, rng.integers(1000, 30522, size=L - 1)].astype(np.int32)]
    rep_ref, z_ref = ob.forward(ids)
    stats(f"base L={L} rep", gb.rep(ids), rep_ref); stats(f"base L={L} logits", gb.logits(ids), z_ref)

"""Diagnostic: engine vs float64 oracle at batch-1 for the large (H=1024) and base (H=768) students
by length and seed (prints the logit error relative to max|logit| and to the per-student pooled
representation; no asserts). Run once per SP_ATTN_TC setting to separate attention from the rest."""
import sys

import numpy as np

sys.path.insert(0, ".")
from oracle.bert import OracleBertGroup  # noqa: E402
from paper_2408_12526_b200 import PRESETS, StudentGroup, random_bert_group  # noqa: E402

for name in ("large", "base"):
    cfg, _ = PRESETS[name]
    for seed in (31, 32, 33):
        w = random_bert_group(cfg, 2, seed=seed)
        g = StudentGroup(w, max_tokens=512, max_seqs=1)
        o = OracleBertGroup(w)
        for L in (128, 384, 512):
            ids = np.r_[101, np.random.default_rng(L + seed).integers(1000, 30522, size=L - 1)].astype(np.int32)
            rep_ref, z_ref = o.forward([ids], 1)
            rep = g.rep(ids, 1)
            z = g.logits(ids)
            _, z2 = o.forward([ids])
            drep = np.abs(rep - rep_ref[0]).max() / np.abs(rep_ref[0]).max()
            dz = np.abs(z - z2[0]).max() / np.abs(z2[0]).max()
            print(f"{name} seed {seed} L={L}: rep0 rel {drep:.2e}  logits rel {dz:.2e}  |z| {np.abs(z2[0]).max():.3f}",
                  flush=True)

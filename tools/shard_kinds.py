"""Per-kernel-kind event-timed breakdown of one shard's batch-1 request (rank 0 of world W) at a few
lengths; events around every launch add ~6 us each, so compare kinds and worlds, not absolutes.

    python tools/shard_kinds.py [W ...]
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2408_12526_b200 import PRESETS  # noqa: E402
from paper_2408_12526_b200.parallel import ShardedStudentGroup  # noqa: E402


def main():
    worlds = [int(a) for a in sys.argv[1:]] or [1, 8]
    cfg, K = PRESETS["base"]
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    ids = torch.from_numpy(np.random.default_rng(0).integers(1000, cfg.vocab, size=512).astype(np.int32)).cuda()
    for w in worlds:
        sh = ShardedStudentGroup(cfg, K, seed=0, rank=0, world=w, max_tokens=512, max_seqs=1)
        logits = torch.empty((1, cfg.n_classes), device="cuda")
        sh.local.set_profiling(True)
        for L in (16, 64, 256, 512):
            cu = torch.tensor([0, L], dtype=torch.int32, device="cuda")
            agg = {}
            for rep in range(12):
                flush.fill_(0.0)
                sh.forward_packed_device(ids, cu, 1, L, L, K, logits, graph=False)
                torch.cuda.synchronize()
                if rep < 2:
                    continue
                for r in sh.local.profile_records():
                    agg[r["kind"]] = agg.get(r["kind"], 0.0) + r["ms"] * 1e3 / 10
            tot = sum(agg.values())
            print(f"world {w} L={L:3d} sum {tot:6.1f} us  " +
                  "  ".join(f"{k} {v:.1f}" for k, v in sorted(agg.items())), flush=True)
        sh.local.set_profiling(False)


if __name__ == "__main__":
    main()

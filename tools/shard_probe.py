"""Batch-1 latency of ONE shard of the base group (rank 0 of world W, no collective) on one GPU:
eager PDL-chained launches vs bucket-graph replay, L ~ U{16..512}, L2 flushed before every request.
Answers whether the N-GPU bench step is host-launch-bound once each GPU holds K/W students.

    python tools/shard_probe.py [W ...]
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2408_12526_b200 import PRESETS  # noqa: E402
from paper_2408_12526_b200.parallel import ShardedStudentGroup  # noqa: E402


def main():
    worlds = [int(a) for a in sys.argv[1:]] or [1, 2, 4, 8]
    cfg, K = PRESETS["base"]
    rng = np.random.default_rng(0)
    lens = rng.integers(16, 513, size=300)
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    for w in worlds:
        sh = ShardedStudentGroup(cfg, K, seed=0, rank=0, world=w, max_tokens=512, max_seqs=1)
        logits = torch.empty((1, cfg.n_classes), device="cuda")
        ids = torch.from_numpy(rng.integers(1000, cfg.vocab, size=512).astype(np.int32)).cuda()
        cus = [torch.tensor([0, int(L)], dtype=torch.int32, device="cuda") for L in lens]
        for t in range(16, 528, 16):  # capture every bucket first
            sh.local.forward_graph_device(ids, torch.tensor([0, t], dtype=torch.int32, device="cuda"), t,
                                          sh.local_k(K), logits)
        res = {}
        for mode in ("eager", "graph"):
            ts = []
            for i, L in enumerate(lens):
                flush.fill_(0.0)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                sh.forward_packed_device(ids, cus[i], 1, int(L), int(L), K, logits, graph=(mode == "graph"))
                e1.record()
                e1.synchronize()
                ts.append(e0.elapsed_time(e1) * 1e3)
            res[mode] = ts[20:]
        print(f"world {w}: {len(sh.students)} student(s)/GPU  eager mean {np.mean(res['eager']):.1f} us "
              f"p50 {np.median(res['eager']):.1f}  graph mean {np.mean(res['graph']):.1f} us "
              f"p50 {np.median(res['graph']):.1f}", flush=True)


if __name__ == "__main__":
    main()

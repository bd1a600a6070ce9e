"""Per-kernel device time of one batch-1 request (CUDA events around every launch), by length."""
import sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_2408_12526_b200 import PRESETS, StudentGroup, random_bert_group
cfg, K = PRESETS[sys.argv[2] if len(sys.argv) > 2 else "base"]
g = StudentGroup(random_bert_group(cfg, K, seed=0), max_tokens=512, max_seqs=1)
fw = torch.empty(256 << 18, device="cuda"); fr = torch.ones(256 << 18, device="cuda")
logits = torch.empty(1, 2, device="cuda")
for L in [int(x) for x in sys.argv[1].split(",")]:
    ids = torch.randint(1000, 30000, (L,), dtype=torch.int32, device="cuda")
    cu = torch.tensor([0, L], dtype=torch.int32, device="cuda")
    run = lambda: g.forward_packed_device(ids, cu, 1, L, L, K, None, logits)
    for _ in range(3): run()
    g.set_profiling(True)
    acc = {}
    for _ in range(10):
        fw.zero_(); fr.sum(); torch.cuda.synchronize()
        run(); torch.cuda.synchronize()
        for i, r in enumerate(g.profile_records()):
            acc.setdefault((i, r["kind"]), []).append(r["ms"] * 1e3)
    g.set_profiling(False)
    tot = sum(np.median(v) for v in acc.values())
    print(f"L={L}: sum of per-launch medians {tot:.1f} us")
    for (i, kind), v in sorted(acc.items()):
        print(f"   {i:2d} {kind:10s} {np.median(v):7.1f}")

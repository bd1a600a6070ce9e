"""Run a few batch-1 requests at fixed lengths (for ncu launch lists)."""
import sys, torch
sys.path.insert(0, ".")
from paper_2408_12526_b200 import PRESETS, StudentGroup, random_bert_group
cfg, K = PRESETS[sys.argv[1] if len(sys.argv) > 1 else "base"]
lens = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "16,512").split(",")]
w = random_bert_group(cfg, K, seed=0)
g = StudentGroup(w, max_tokens=max(lens), max_seqs=1)
logits = torch.empty(1, 2, device="cuda")
for L in lens:
    ids = torch.randint(1000, 30000, (L,), dtype=torch.int32, device="cuda")
    cu = torch.tensor([0, L], dtype=torch.int32, device="cuda")
    for _ in range(2):
        g.forward_packed_device(ids, cu, 1, L, L, K, None, logits)
torch.cuda.synchronize()
print("ok")

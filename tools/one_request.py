"""Run a few batch-1 requests of one length (for ncu captures of individual kernels)."""
import sys, torch
sys.path.insert(0, ".")
from paper_2408_12526_b200 import PRESETS, StudentGroup, random_bert_group
cfg, K = PRESETS[sys.argv[2] if len(sys.argv) > 2 else "base"]
L = int(sys.argv[1])
g = StudentGroup(random_bert_group(cfg, K, seed=0), max_tokens=512, max_seqs=1)
ids = torch.randint(1000, 30000, (L,), dtype=torch.int32, device="cuda")
cu = torch.tensor([0, L], dtype=torch.int32, device="cuda")
logits = torch.empty(1, 2, device="cuda")
fw = torch.empty(256 << 18, device="cuda"); fr = torch.ones(256 << 18, device="cuda")
for _ in range(int(sys.argv[3]) if len(sys.argv) > 3 else 3):
    fw.zero_(); fr.sum()
    g.forward_packed_device(ids, cu, 1, L, L, K, None, logits)
torch.cuda.synchronize()
print("ok")

"""forward_host latency of the FIRST request of each 16-token bucket after prepare_graphs vs a repeat."""
import sys, time, numpy as np, torch
sys.path.insert(0, ".")
from paper_2408_12526_b200 import PRESETS, StudentGroup, random_bert_group
cfg, K = PRESETS["base"]
g = StudentGroup(random_bert_group(cfg, K, seed=0), max_tokens=512, max_seqs=1)
g.prepare_graphs(512, K)
fw = torch.empty(256 << 18, device="cuda"); fr = torch.ones(256 << 18, device="cuda")
out = np.empty((1, 2), np.float32)
first, again = [], []
for L in range(24, 512, 32):
    ids = torch.randint(1000, 30000, (L,), dtype=torch.int32).pin_memory().numpy()
    cu = torch.tensor([0, L], dtype=torch.int32).pin_memory().numpy()
    for lst in (first, again):
        fw.zero_(); fr.sum(); torch.cuda.synchronize()
        t0 = time.perf_counter(); g.forward_host(ids, cu, K, out=out); lst.append(time.perf_counter() - t0)
d = 1e6 * (np.array(first) - np.array(again))
print(f"first call - repeat over {len(d)} buckets: median {np.median(d):.1f} us, max {d.max():.1f} us; "
      f"first median {1e6 * np.median(first):.1f} us")

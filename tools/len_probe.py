"""Batch-1 graph-replay latency (L2 flushed) at many lengths: compare engine knobs via env."""
import os, sys, numpy as np, torch
sys.path.insert(0, ".")
if os.environ.get("SP_LIB_OVERRIDE"):  # A/B another build of the engine library
    from pathlib import Path
    import paper_2408_12526_b200._lib as _L
    _L.LIB_PATH = Path(os.environ["SP_LIB_OVERRIDE"])
from paper_2408_12526_b200 import PRESETS, StudentGroup, random_bert_group
cfg, K = PRESETS[os.environ.get("PRESET", "base")]
g = StudentGroup(random_bert_group(cfg, K, seed=0), max_tokens=512, max_seqs=1)
fw = torch.empty(256 << 18, device="cuda"); fr = torch.ones(256 << 18, device="cuda")
logits = torch.empty(1, 2, device="cuda")
out = []
for L in [int(x) for x in sys.argv[1].split(",")]:
    ids = torch.randint(1000, 30000, (L,), dtype=torch.int32, device="cuda")
    cu = torch.tensor([0, L], dtype=torch.int32, device="cuda")
    run = lambda: g.forward_packed_device(ids, cu, 1, L, L, K, None, logits)
    for _ in range(3): run()
    s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s): run()
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph): run()
    ts = []
    for _ in range(60):
        if not os.environ.get("NO_FLUSH"):
            fw.zero_(); fr.sum()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); graph.replay(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1) * 1e3)
    ts = np.sort(ts)[6:-6]  # trimmed mean: the event clock ticks in ~2 us steps, a median stays on a tick
    out.append(f"{L}:{ts.mean():.1f}")
print(" ".join(out))

"""How much of a batch-1 request is host launch overhead? Eager vs CUDA-graph replay."""
import sys, numpy as np, torch
sys.path.insert(0, ".")
import os
if os.environ.get("SP_LIB_OVERRIDE"):  # A/B another build of the engine library
    from pathlib import Path
    import paper_2408_12526_b200._lib as _L
    _L.LIB_PATH = Path(os.environ["SP_LIB_OVERRIDE"])
from paper_2408_12526_b200 import PRESETS, StudentGroup, random_bert_group
cfg, K = PRESETS["base"]
w = random_bert_group(cfg, K, seed=0)
g = StudentGroup(w, max_tokens=512, max_seqs=1)
fw = torch.empty(256 << 18, device="cuda"); fr = torch.ones(256 << 18, device="cuda")
def flush(): fw.zero_(); fr.sum()
logits = torch.empty(1, 2, device="cuda")
for L in (16, 64, 128, 256, 512):
    ids = torch.randint(1000, 30000, (L,), dtype=torch.int32, device="cuda")
    cu = torch.tensor([0, L], dtype=torch.int32, device="cuda")
    run = lambda: g.forward_packed_device(ids, cu, 1, L, L, K, None, logits)
    for _ in range(3): run()
    torch.cuda.synchronize()
    def timeit(fn, n=20):
        ts = []
        for _ in range(n):
            flush(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1) * 1e3)
        return np.median(ts)
    eager = timeit(run)
    s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        run()
    torch.cuda.synchronize()
    with torch.cuda.graph(graph):
        run()
    gr = timeit(graph.replay)
    # back-to-back without flush (L2-warm upper bound)
    nof = []
    for _ in range(20):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); graph.replay(); e1.record(); torch.cuda.synchronize(); nof.append(e0.elapsed_time(e1) * 1e3)
    wb = 236.4e6
    print(f"L={L:4d} eager={eager:7.1f}us graph={gr:7.1f}us ({wb/gr/1e3/6533.8*100:4.1f}% HBM) graph_l2warm={np.median(nof):7.1f}us")

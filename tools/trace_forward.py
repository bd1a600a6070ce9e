"""Absolute timeline of every GEMM CTA in one batch-1 forward (PDL overlap visible)."""
import sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_2408_12526_b200 import PRESETS, StudentGroup, random_bert_group, _lib
import os
cfg, K = PRESETS[os.environ.get("PRESET", "base")]
w = random_bert_group(cfg, K, seed=0)
g = StudentGroup(w, max_tokens=512, max_seqs=1)
lib = _lib.load()
fw = torch.empty(256 << 18, device="cuda"); fr = torch.ones(256 << 18, device="cuda")
logits = torch.empty(1, 2, device="cuda")
tr = torch.zeros(8 * 20000, dtype=torch.int64, device="cuda")
def names_for(L):  # GEMM launches in order (current bert_forward; the fused MLP and attention are not traced)
    mid = ["qkv", "o", "ffn1", "ffn2"] if not (129 <= L < 256) else ["qkv", "o"]
    last = ["kv", "q_cls"] if L >= 256 else ["qkv"]
    return mid + last + ["o_cls", "ffn1c", "ffn2c", "pool"]
for L in [int(x) for x in sys.argv[1].split(",")]:
    ids = torch.randint(1000, 30000, (L,), dtype=torch.int32, device="cuda")
    cu = torch.tensor([0, L], dtype=torch.int32, device="cuda")
    run = lambda: g.forward_packed_device(ids, cu, 1, L, L, K, None, logits)
    for _ in range(3): run()
    torch.cuda.synchronize()
    lib.sp_debug_set_gemm_trace(tr.data_ptr())
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        run()
    import ctypes
    cnt = (ctypes.c_int32 * 64)()
    sizes = list(cnt[:lib.sp_debug_gemm_trace_launches(cnt, 64)])
    lib.sp_debug_set_gemm_trace(None)
    for _ in range(3): graph.replay()
    fw.zero_(); fr.sum(); torch.cuda.synchronize()
    tr.zero_()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); graph.replay(); e1.record(); torch.cuda.synchronize()
    t = tr.view(-1, 8).cpu().numpy().astype(np.float64)
    base = t[t[:, 0] > 0][:, 0].min()
    off = 0
    print(f"L={L}: event {e0.elapsed_time(e1)*1e3:.1f} us")
    gi = 0
    for li, n in enumerate(sizes):
        names = names_for(L)
        aux = n < 0
        kind = (-n) // 100000 if aux else 0
        n = (-n) % 100000 if aux else n
        if aux:
            nm = {1: "ln", 2: "attn"}.get(kind, "aux")
        else:
            nm = names[gi] if gi < len(names) else f"g{gi}"
            gi += 1
        raw = t[off:off + n]; off += n
        raw = raw[raw[:, 0] > 0]
        seg = (raw - base) / 1e3
        if len(seg) == 0:
            continue
        if aux:
            if kind == 2:  # attention: entry, dep, S issued, scores seen, last PV issued, PV done, end
                med = lambda c: np.median(seg[raw[:, c] > 0][:, c]) if (raw[:, c] > 0).any() else -1
                print(f"  {nm:5s} ctas={n:4d} entry[{seg[:,0].min():6.1f},{seg[:,0].max():6.1f}] dep={med(1):6.1f} "
                      f"s0={med(2):6.1f} scores={med(3):6.1f} pv_issued={med(4):6.1f} pv_done={med(5):6.1f} "
                      f"end={seg[raw[:, 7] > 0][:, 7].max():6.1f}")
                continue
            live = seg[raw[:, 3] > 0]
            print(f"  {nm:5s} ctas={n:4d} entry[{seg[:,0].min():6.1f},{seg[:,0].max():6.1f}] "
                  f"dep={np.median(live[:,3]) if len(live) else -1:6.1f} end={live[:,7].max() if len(live) else -1:6.1f}")
            continue
        print(f"  {nm:5s} ctas={n:4d} entry[{seg[:,0].min():6.1f},{seg[:,0].max():6.1f}] wpre={np.median(seg[:,2]):6.1f} mma0={np.median(seg[:,4]):6.1f} "
              f"dep={np.median(seg[:,3]):6.1f} last_commit={seg[:,5].max():6.1f} epi0_max={seg[:,6].max():6.1f} end={seg[:,7].max():6.1f}")

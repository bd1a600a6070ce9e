"""Per-CTA timeline of the grouped GEMM at batch-1 B8 shapes (debug trace hook)."""
import sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_2408_12526_b200 import _lib
lib = _lib.load()
G, T = 8, int(sys.argv[1]) if len(sys.argv) > 1 else 224
shapes = {"qkv": (2304, 768, 1, 0), "o": (768, 768, 3, 0), "ffn1": (3072, 768, 1, 2), "ffn2": (768, 3072, 3, 0)}
import os
if os.environ.get("TRACE_SHAPES") == "epi":
    shapes = {"ffn1_id": (3072, 768, 1, 0), "ffn1_gelu": (3072, 768, 1, 2), "qkv_gelu": (2304, 768, 1, 2),
              "n1536_gelu": (1536, 768, 1, 2), "ffn1_G4": (3072, 768, 1, 2)}
flush = torch.empty(256 << 18, device="cuda")
flush_r = torch.ones(256 << 18, device="cuda")
def do_flush():
    flush.zero_(); flush_r.sum()
for name, (N, K, splits, act) in shapes.items():
    G = 4 if name.endswith("_G4") else 8
    w = (torch.randn(G, N, K, device="cuda") * 0.02).half()
    x = torch.randn(G * 512, K, device="cuda").half()
    out = torch.empty(splits, G, 512, N, device="cuda", dtype=torch.float32)
    bias = torch.zeros(G, N, device="cuda")
    tr = torch.zeros(8 * 8192, dtype=torch.int64, device="cuda")
    def run():
        _lib.check(lib.sp_op_gemm(w.data_ptr(), x.data_ptr(), G, N, K, T, 512, G * 512, bias.data_ptr(), act,
                                  out.data_ptr(), 0 if splits == 1 else 1, splits, None))
    for _ in range(3): run()
    ts = []
    for _ in range(5):
        do_flush(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); run(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1) * 1e3)
    do_flush(); torch.cuda.synchronize()
    lib.sp_debug_set_gemm_trace(tr.data_ptr()); run(); torch.cuda.synchronize()
    import ctypes
    cnt = (ctypes.c_int32 * 4)(); lib.sp_debug_gemm_trace_launches(cnt, 4); n_cta = cnt[0]
    lib.sp_debug_set_gemm_trace(None)
    t = tr.view(-1, 8)[:n_cta].cpu().numpy().astype(np.float64)
    t0 = t[:, 0].min()
    rel = (t - t0) / 1e3
    wbytes = G * N * K * 2
    print(f"{name}: N={N} K={K} splits={splits} ctas={n_cta} event_us={np.median(ts):.1f} "
          f"W={wbytes/1e6:.1f}MB -> {wbytes/np.median(ts)/1e3:.0f} GB/s")
    labels = ["entry", "prologue", "tma0", "tma_last", "mma0", "commit_last", "epi0", "exit"]
    for i, l in enumerate(labels):
        c = rel[:, i]
        print(f"   {l:12s} min={c.min():7.2f} med={np.median(c):7.2f} max={c.max():7.2f} us")

"""Persistent GEMM at a batched shape: where does the MMA thread wait (operands vs accumulators)?"""
import sys, os, ctypes, numpy as np, torch
sys.path.insert(0, ".")
from paper_2408_12526_b200 import _lib
lib = _lib.load()
G = int(os.environ.get("TP_G", 8)); T = int(sys.argv[1]) if len(sys.argv) > 1 else 512
H = int(os.environ.get("TP_H", 768))
shapes = {"qkv": (3 * H, H, 0), "o": (H, H, 0), "ffn1_gelu": (4 * H, H, 2), "ffn1_id": (4 * H, H, 0),
          "ffn2": (H, 4 * H, 0)}
flush = torch.empty(256 << 18, device="cuda"); flush_r = torch.ones(256 << 18, device="cuda")
for name, (N, K, act) in shapes.items():
    w = (torch.randn(G, N, K, device="cuda") * 0.02).half()
    x = torch.randn(G * T, K, device="cuda").half()
    xl = (torch.randn(G * T, K, device="cuda") * 1e-4).half()  # (hi, lo) operand as the engine runs it
    out = torch.empty(G, T, N, device="cuda", dtype=torch.float16)
    bias = torch.zeros(G, N, device="cuda")
    tr = torch.zeros(8 * 4096, dtype=torch.int64, device="cuda")
    run = lambda: _lib.check(lib.sp_op_gemm(w.data_ptr(), x.data_ptr(), xl.data_ptr(), G, N, K, T, T, G * T,
                                            bias.data_ptr(), act, out.data_ptr(), None, 0, 1, None))
    for _ in range(3): run()
    ts = []
    for _ in range(5):
        if not os.environ.get("NO_FLUSH"): flush.zero_(); flush_r.sum()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); run(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1) * 1e3)
    if not os.environ.get("NO_FLUSH"): flush.zero_(); flush_r.sum()
    torch.cuda.synchronize()
    lib.sp_debug_set_gemm_trace(tr.data_ptr()); run(); torch.cuda.synchronize()
    cnt = (ctypes.c_int32 * 4)(); lib.sp_debug_gemm_trace_launches(cnt, 4); n_cta = cnt[0]
    lib.sp_debug_set_gemm_trace(None)
    t = tr.view(-1, 8)[:n_cta].cpu().numpy().astype(np.float64)
    fl = 2.0 * G * N * K * T * 2  # executed: two MMAs per k-slice
    us = np.median(ts)
    lead = t[t[:, 5] > 0]  # CTAs that issued MMAs
    span = (lead[:, 5] - lead[:, 4]) / 1e3
    print(f"{name}: N={N} K={K} act={act} ctas={n_cta} {us:.1f} us = {fl / us / 1e6:.0f} TFLOP/s; MMA span med {np.median(span):.1f} us; "
          f"MMA waits (med over issuing CTAs): operands {np.median(lead[:, 1]) / 1e3:.1f} us, accumulator {np.median(lead[:, 3]) / 1e3:.1f} us")
    t0 = t[:, 0].min()
    rel = lambda c: (t[:, c][t[:, c] > 0] - t0) / 1e3
    print(f"   timeline (us from first CTA entry, median/max): entry {np.median(rel(0)):.1f}/{rel(0).max():.1f}  "
          f"first MMA {np.median((lead[:, 4] - t0) / 1e3):.1f}  last commit {np.median((lead[:, 5] - t0) / 1e3):.1f}/"
          f"{((lead[:, 5] - t0) / 1e3).max():.1f}  epi start {np.median(rel(6)):.1f}  epi end {np.median(rel(7)):.1f}/{rel(7).max():.1f}")

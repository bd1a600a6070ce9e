"""Per-CTA timeline of the single-pass tcgen05 attention (attn_tc2) at batch-1 shapes.

    python tools/trace_attn.py 256,512
Prints, per length, the kernel span and the median per-CTA phase times (us from CTA entry):
setup, per chunk: scores ready (softmax sees S_j) / P_j published / K,V_j load issued, epilogue, end.
"""
import sys, ctypes, numpy as np, torch
sys.path.insert(0, ".")
from paper_2408_12526_b200 import _lib
lib = _lib.load()
G, NH, D = 8, 12, 64
H = NH * D
for L in [int(x) for x in sys.argv[1].split(",")]:
    qkv = (torch.randn(G, L, 3 * H, device="cuda") * 0.5).half()
    ctx = torch.empty(G, L, H, device="cuda").half()
    cu = torch.tensor([0, L], dtype=torch.int32, device="cuda")
    n_cta = G * NH * ((L + 127) // 128)
    tr = torch.zeros(n_cta * 16, dtype=torch.int64, device="cuda")
    run = lambda: _lib.check(lib.sp_op_attention(qkv.data_ptr(), ctx.data_ptr(), cu.data_ptr(), 1, L, G, NH, D, L, None))
    for _ in range(3): run()
    lib.sp_debug_set_attn_trace(ctypes.c_void_p(tr.data_ptr()))
    torch.cuda.synchronize(); run(); torch.cuda.synchronize()
    lib.sp_debug_set_attn_trace(None)
    t = tr.view(n_cta, 16).cpu().numpy().astype(np.float64)
    t = t[t[:, 0] > 0]
    base = t[:, 0].min()
    rel = lambda c: (t[:, c] - t[:, 0]) / 1e3
    print(f"L={L}: {len(t)} CTAs, span {(t[:, 15].max() - base) / 1e3:.1f} us; CTA entry spread "
          f"{(t[:, 0].max() - base) / 1e3:.1f} us; per-CTA duration p50 {np.median(rel(15)):.2f} max {rel(15).max():.2f}")
    nch = (L + 127) // 128
    print(f"   setup {np.median(rel(1)):.2f}  " + "  ".join(
        f"c{j}: load {np.median(rel(10 + j)):.2f} S {np.median(rel(2 + j)):.2f} P {np.median(rel(6 + j)):.2f}"
        for j in range(min(nch, 4))) + f"  epi {np.median(rel(14)):.2f} end {np.median(rel(15)):.2f}")

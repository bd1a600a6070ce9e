import sys, torch
sys.path.insert(0, ".")
from paper_2408_12526_b200 import _lib
lib = _lib.load()
for (N, K, T, G) in [(256, 64, 160, 1), (256, 128, 160, 1), (512, 64, 160, 1)]:
    torch.manual_seed(0)
    w = (torch.randn(G, N, K, device="cuda") * 0.05).half(); x = torch.randn(G * T, K, device="cuda").half()
    out = torch.zeros(G, T, N, device="cuda"); bias = torch.zeros(G, N, device="cuda")
    _lib.check(lib.sp_op_gemm(w.data_ptr(), x.data_ptr(), G, N, K, T, T, G * T, bias.data_ptr(), 0, out.data_ptr(), 1, 1, None))
    torch.cuda.synchronize()
    ref = torch.stack([x[g*T:(g+1)*T].float() @ w[g].float().T for g in range(G)])
    bad = ((out - ref).abs() > 1e-2)
    rows = bad.any(dim=2)[0].nonzero().flatten().tolist(); cols = bad.any(dim=1)[0].nonzero().flatten().tolist()
    print((N, K, T, G), "bad tokens", rows[:5], "...", len(rows), "bad feats", cols[:3], "...", cols[-3:] if cols else [], len(cols), flush=True)

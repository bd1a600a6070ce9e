"""One grouped GEMM launch of a given shape (for ncu): gemm_one.py N K T splits act [G]."""
import sys, torch
sys.path.insert(0, ".")
from paper_2408_12526_b200 import _lib
lib = _lib.load()
N, K, T, splits, act = (int(a) for a in sys.argv[1:6])
G = int(sys.argv[6]) if len(sys.argv) > 6 else 8
w = (torch.randn(G, N, K, device="cuda") * 0.02).half()
x = torch.randn(2, G * 512, K, device="cuda").half()  # (hi, lo) operand terms
out = torch.empty(splits, G, 512, N, device="cuda", dtype=torch.float32)
bias = torch.zeros(G, N, device="cuda")
for _ in range(4):
    _lib.check(lib.sp_op_gemm(w.data_ptr(), x[0].data_ptr(), x[1].data_ptr(), G, N, K, T, 512, G * 512,
                              bias.data_ptr(), act, out.data_ptr(), None, 1, splits, None))
torch.cuda.synchronize()
print("ok")

import sys, os, subprocess
sys.path.insert(0, ".")
shapes = [(256, 192, 256, 3), (256, 192, 300, 3), (2304, 768, 256, 8), (768, 768, 512, 8), (3072, 768, 512, 8)]
code = r'''
import sys, torch; sys.path.insert(0, ".")
from paper_2408_12526_b200 import _lib
lib = _lib.load()
N, K, T, G = %d, %d, %d, %d
w = (torch.randn(G, N, K, device="cuda") * 0.05).half(); x = torch.randn(G * T, K, device="cuda").half()
out = torch.empty(G, T, N, device="cuda"); bias = torch.zeros(G, N, device="cuda")
_lib.check(lib.sp_op_gemm(w.data_ptr(), x.data_ptr(), G, N, K, T, T, G * T, bias.data_ptr(), 0, out.data_ptr(), 1, 1, None))
torch.cuda.synchronize()
ref = torch.stack([x[g*T:(g+1)*T].float() @ w[g].float().T for g in range(G)])
print("maxerr", (out - ref).abs().max().item())
'''
for sh in shapes:
    r = subprocess.run([sys.executable, "-c", code % sh], capture_output=True, text=True, timeout=60,
                       env={**os.environ, "SP_PERSIST_PAIR": "1"})
    print(sh, r.returncode, (r.stdout.strip() or r.stderr.strip().splitlines()[-1])[:150], flush=True)

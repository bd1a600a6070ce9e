"""End-to-end batch-1 latency through StudentGroup.forward_host (host ids in, logits out), by length."""
import os, sys, time, numpy as np, torch
sys.path.insert(0, ".")
if os.environ.get("SP_LIB_OVERRIDE"):  # A/B another build of the engine library
    from pathlib import Path
    import paper_2408_12526_b200._lib as _L
    _L.LIB_PATH = Path(os.environ["SP_LIB_OVERRIDE"])
from paper_2408_12526_b200 import PRESETS, StudentGroup, random_bert_group
cfg, K = PRESETS["base"]
g = StudentGroup(random_bert_group(cfg, K, seed=0), max_tokens=512, max_seqs=1)
g.prepare_graphs(512, K)
fw = torch.empty(256 << 18, device="cuda"); fr = torch.ones(256 << 18, device="cuda")
out = np.empty((1, 2), np.float32)
for L in (16, 128, 512):
    ids = torch.randint(1000, 30000, (L,), dtype=torch.int32).pin_memory().numpy()
    cu = torch.tensor([0, L], dtype=torch.int32).pin_memory().numpy()
    for _ in range(5): g.forward_host(ids, cu, K, out=out)
    ts = []
    for _ in range(50):
        fw.zero_(); fr.sum(); torch.cuda.synchronize()
        t0 = time.perf_counter(); g.forward_host(ids, cu, K, out=out); ts.append(time.perf_counter() - t0)
    print(f"L={L:4d} e2e p50 {1e6 * np.median(ts):7.1f} us")

# host-side breakdown at L=16: Python wrapper vs raw C call vs empty-ish calls
import ctypes
L = 16
ids = torch.randint(1000, 30000, (L,), dtype=torch.int32).pin_memory().numpy()
cu = torch.tensor([0, L], dtype=torch.int32).pin_memory().numpy()
h, lib = g._handle, g._lib
sh = torch.cuda.current_stream().cuda_stream
args = (h, ids.ctypes.data, cu.ctypes.data, 1, L, K, out.ctypes.data, 1, sh)
def timeit(fn, n=200):
    ts = []
    for _ in range(n):
        t0 = time.perf_counter(); fn(); ts.append(time.perf_counter() - t0)
    return 1e6 * np.median(ts)
print(f"wrapper forward_host     {timeit(lambda: g.forward_host(ids, cu, K, out=out)):7.1f} us (no flush, L2 warm)")
print(f"raw sp_group_forward_host {timeit(lambda: lib.sp_group_forward_host(*args)):7.1f} us")
print(f"local_k                   {timeit(lambda: g.local_k(K)):7.1f} us")
print(f"stream handle             {timeit(lambda: torch.cuda.current_stream().cuda_stream):7.1f} us")
print(f"torch sync (idle)         {timeit(lambda: torch.cuda.synchronize()):7.1f} us")
# the same call through the PyTorch C++ extension (torch.ops.studentpar.group_forward_host)
from paper_2408_12526_b200 import _lib as _L2
torch.ops.load_library(str(_L2.TORCH_LIB_PATH))
ids_t, cu_t, out_t = torch.from_numpy(ids), torch.from_numpy(cu), torch.from_numpy(out)
op = torch.ops.studentpar.group_forward_host
print(f"torch op forward_host     {timeit(lambda: op(h.value, ids_t, cu_t, K, out_t, True, 0)):7.1f} us")
print(f"torch op (from numpy)     {timeit(lambda: op(h.value, torch.from_numpy(ids), torch.from_numpy(cu), K, torch.from_numpy(out), True, 0)):7.1f} us")

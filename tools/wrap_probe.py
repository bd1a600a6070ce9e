import sys, time, numpy as np, torch, ctypes as C
sys.path.insert(0, ".")
from paper_2408_12526_b200 import PRESETS, StudentGroup, random_bert_group
cfg, K = PRESETS["base"]
g = StudentGroup(random_bert_group(cfg, K, seed=0), max_tokens=512, max_seqs=1)
g.prepare_graphs(64, K)
L = 16
ids = torch.randint(1000, 30000, (L,), dtype=torch.int32).pin_memory().numpy()
cu = np.array([0, L], np.int32)
out = np.empty((1, 2), np.float32)
def timeit(fn, n=300):
    for _ in range(20): fn()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter(); fn(); ts.append(time.perf_counter() - t0)
    return 1e6 * np.median(ts)
h, lib = g._handle, g._lib
raw = lambda: lib.sp_group_forward_host(h, ids.ctypes.data, cu.ctypes.data, 1, L, K, out.ctypes.data, 1,
                                         torch._C._cuda_getCurrentRawStream(0))
print(f"wrapper forward_host          {timeit(lambda: g.forward_host(ids, cu, K, out=out)):7.1f} us")
print(f"ctypes + _cuda_getCurrentRawStream {timeit(raw):7.1f} us")
print(f"_cuda_getCurrentRawStream alone {timeit(lambda: torch._C._cuda_getCurrentRawStream(0)):7.2f} us")
print(f"ascontiguousarray x2          {timeit(lambda: (np.ascontiguousarray(ids, dtype=np.int32), np.ascontiguousarray(cu, dtype=np.int32))):7.2f} us")
print(f"from_numpy x3                 {timeit(lambda: (torch.from_numpy(ids), torch.from_numpy(cu), torch.from_numpy(out))):7.2f} us")
print(f"local_k                       {timeit(lambda: g.local_k(K)):7.2f} us")

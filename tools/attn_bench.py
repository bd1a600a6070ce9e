"""Op-level attention timing (batch-1 shapes): K students x heads over one sequence of L tokens."""
import os, sys, numpy as np, torch
sys.path.insert(0, ".")
if os.environ.get("SP_LIB_OVERRIDE"):  # A/B another build of the engine library
    from pathlib import Path
    import paper_2408_12526_b200._lib as _L
    _L.LIB_PATH = Path(os.environ["SP_LIB_OVERRIDE"])
from paper_2408_12526_b200 import _lib
lib = _lib.load()
G, NH, D = 8, 12, 64
H = NH * D
for L in [int(x) for x in sys.argv[1].split(",")]:
    qkv = (torch.randn(G, L, 3 * H, device="cuda") * 0.5).half()
    ctx = torch.empty(2, G, L, H, device="cuda").half()  # (hi, lo) context planes
    cu = torch.tensor([0, L], dtype=torch.int32, device="cuda")
    run = lambda: _lib.check(lib.sp_op_attention(qkv.data_ptr(), ctx[0].data_ptr(), ctx[1].data_ptr(), cu.data_ptr(), 1, L, G, NH, D, L,
                                                         None))
    for _ in range(3): run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50): run()
    e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / 50
    fl = 4.0 * G * NH * L * L * D
    print(f"L={L}: {us:.1f} us/launch ({fl / us / 1e6:.0f} TFLOP/s)")

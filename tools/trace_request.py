"""Timeline of the whole-request persistent kernel: per-stage completion stamps across CTAs."""
import sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_2408_12526_b200 import PRESETS, StudentGroup, random_bert_group, _lib
preset = sys.argv[2] if len(sys.argv) > 2 else "base"
cfg, K = PRESETS[preset]
w = random_bert_group(cfg, K, seed=0)
g = StudentGroup(w, max_tokens=512, max_seqs=4)
lib = _lib.load()
nsm = torch.cuda.get_device_properties(0).multi_processor_count
tr = torch.zeros(128 * nsm, dtype=torch.int64, device="cuda")
fw = torch.empty(256 << 18, device="cuda"); fr = torch.ones(256 << 18, device="cuda")
logits = torch.empty(1, 2, device="cuda")
names = ["embed"] + [f"L{l}.{s}" for l in range(cfg.n_layers) for s in ("qkv", "attn", "o", "ln1", "ffn1", "ffn2", "ln2")] + ["pool", "head"]
check = "--check" in sys.argv
for L in [int(x) for x in sys.argv[1].split(",")]:
    rng = np.random.default_rng(L)
    ids_np = np.r_[101, rng.integers(1000, 30000, size=L - 1)].astype(np.int32)
    ids = torch.tensor(ids_np, device="cuda")
    cu = torch.tensor([0, L], dtype=torch.int32, device="cuda")
    run = lambda: g.forward_packed_device(ids, cu, 1, L, L, K, None, logits)
    for _ in range(3): run()
    torch.cuda.synchronize()
    ts = []
    for _ in range(20):
        fw.zero_(); fr.sum()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); run(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1) * 1e3)
    lib.sp_debug_set_request_trace(tr.data_ptr())
    tr.zero_(); fw.zero_(); fr.sum(); torch.cuda.synchronize()
    run(); torch.cuda.synchronize()
    lib.sp_debug_set_request_trace(None)
    t = tr.view(nsm, 128).cpu().numpy().astype(np.float64)
    base = t[:, 0].min()
    rel = (t[:, :64] - base) / 1e3
    print(f"L={L}: event median {np.median(ts):.1f} us; launches {g.last_launches}")
    for i, nm in enumerate(names):
        col = rel[:, 1 + i]
        print(f"  {nm:9s} min {col.min():7.1f} med {np.median(col):7.1f} max {col.max():7.1f}")
    nph = 4 * cfg.n_layers + 1
    wp = rel[:, 40:40 + nph]
    print("  W-producer issue-done per phase (max over CTAs):", " ".join(f"{x:.1f}" for x in wp.max(0)))
    xd = rel[:, 20:20 + nph]; mm = rel[:, 52:52 + nph]
    print("  X first-dep met per phase (min/med/max):", " | ".join(f"{a:.1f}/{b:.1f}/{c:.1f}" for a, b, c in zip(xd.min(0), np.median(xd, 0), xd.max(0))))
    print("  MMA phase done (min/med/max):          ", " | ".join(f"{a:.1f}/{b:.1f}/{c:.1f}" for a, b, c in zip(mm.min(0), np.median(mm, 0), mm.max(0))))
    acc = t[:, 64:64 + 5 * nph].reshape(nsm, nph, 5) / 1e3
    print("  epilogue step time, us (median over CTAs): phase: accwait tmem->glob arrive fixup signal")
    for ph in range(nph):
        m_ = np.median(acc[:, ph, :], 0); mx = acc[:, ph, :].max(0)
        print(f"    {ph}: " + " ".join(f"{a:6.2f}" for a in m_) + "   max " + " ".join(f"{a:6.2f}" for a in mx))
    if check:
        from oracle.bert import OracleBertGroup
        _, zr = OracleBertGroup(w).forward([ids_np], K)
        z = logits.double().cpu().numpy()
        print("  logits", z.ravel(), "oracle", zr.ravel(), "rel err", float(np.abs(z - zr).max() / np.abs(zr).max()))

"""Parity seed sweep (GPU + CPU oracle): the engine vs the float64 oracle on UNSELECTED seeds at every
north-star configuration at full K, batch-1, L in {16, 128, 384, 512}; every prefix k is checked
from the same per-student pooled outputs.

    python tools/parity_sweep.py [--seeds 10] [--first-seed 100] [--configs base,large,k32] > profiles/r2_parity_seed_sweep.txt

Bar: max over rows of |dz| / max|z_ref| <= 1e-3 (tests/conftest.rel_err_rows), identical argmax where
the top-2 margin exceeds twice that. The oracle (oracle/bert.py) is the checker only; its students
run in parallel worker processes (one BLAS thread each).
"""
import argparse
import os
import sys
import time
from multiprocessing import get_context

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
import numpy as np  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

_W = None  # weights of the current (config, seed), inherited by forked workers


def _pooled(job):
    from oracle.bert import OracleBertGroup

    m, ids = job
    return OracleBertGroup(_W).pooled(m, [ids])[0]


def main():
    global _W
    ap = argparse.ArgumentParser()
    ap.add_argument("--seeds", type=int, default=10)
    ap.add_argument("--first-seed", type=int, default=100)
    ap.add_argument("--configs", default="base,large,k32")
    ap.add_argument("--lens", default="16,128,384,512")
    ap.add_argument("--workers", type=int, default=len(os.sched_getaffinity(0)))
    args = ap.parse_args()
    from paper_2408_12526_b200 import PRESETS, StudentGroup, random_bert_group
    from oracle.dense import IDENTITY, dense_layer, ensemble_rep

    lens = [int(x) for x in args.lens.split(",")]
    worst = 0.0
    n_cases = n_fail = 0
    print(f"# tools/parity_sweep.py: seeds {args.first_seed}..{args.first_seed + args.seeds - 1}, L in {lens}, "
          f"batch-1, engine (fp16 weights, (hi, lo) activations) vs float64 oracle; err = max|dz| / max|z_ref|")
    for name in args.configs.split(","):
        cfg, K = PRESETS[name]
        for seed in range(args.first_seed, args.first_seed + args.seeds):
            t0 = time.time()
            _W = random_bert_group(cfg, K, seed=seed)
            grp = StudentGroup(_W, max_tokens=512, max_seqs=1)
            rng = np.random.default_rng(seed)
            reqs = [np.r_[101, rng.integers(1000, cfg.vocab, size=L - 1)].astype(np.int32) for L in lens]
            with get_context("fork").Pool(args.workers) as pool:
                pooled = pool.map(_pooled, [(m, ids) for ids in reqs for m in range(K)])
            wc, bc = _W.w_cls.astype(np.float64), _W.b_cls.astype(np.float64)
            alpha = [float(a) for a in _W.alpha]
            for li, (L, ids) in enumerate(zip(lens, reqs)):
                finals = [pooled[li * K + m][None, :] for m in range(K)]
                errs = []
                for k in range(1, K + 1):
                    z_ref = dense_layer(wc, bc, ensemble_rep(finals, alpha, k), IDENTITY)[0]
                    z = grp.logits(ids, k)
                    err = float(np.abs(z - z_ref).max() / np.abs(z_ref).max())
                    srt = np.sort(z_ref)
                    if srt[-1] - srt[-2] > 2e-3 * np.abs(z_ref).max() and np.argmax(z) != np.argmax(z_ref):
                        err = float("inf")
                    errs.append(err)
                full = errs[-1]
                n_cases += 1
                n_fail += int(max(errs) > 1e-3)
                worst = max(worst, max(errs))
                print(f"{name:5s} K={K:2d} seed {seed} L={L:3d}  full-K err {full:.2e}  worst prefix err "
                      f"{max(errs):.2e} (k={int(np.argmax(errs)) + 1})  {'ok' if max(errs) <= 1e-3 else 'FAIL'}",
                      flush=True)
            grp.close()
            print(f"#   {name} seed {seed}: {time.time() - t0:.0f} s", flush=True)
    print(f"# {n_cases} (config, seed, L) cases x every prefix k: worst error {worst:.2e}, {n_fail} over 1e-3")


if __name__ == "__main__":
    main()

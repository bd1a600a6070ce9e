"""Bursty Poisson trace with adaptive student count on the real engine (BASELINE.json config 4).

The trace has the reference's phase shape (pkg/configs/simulate.json:31-36: 2000 -> 10000 -> 2000
rps) built exactly as cli.py:191-202 builds it (serving.generate_phases), lengths from the
reference's 16-bin histogram scaled to L <= 512. Every request is dispatched immediately on
arrival (no batching wait, no padding) through StudentGroup.forward_host (one C call: H2D ids,
forward, D2H logits); its measured wall time replaces the simulator's analytic service_time
(servesim.py:486). The controller (decide_controller_action, servesim.py:317-342) drops a
trailing student while the backlog is full and adds one back after an idle window; k is
snapshotted per request.

    python tools/serve_bursty.py [--scale 0.2] [--out gpurun_out/serve_bursty.json]
"""
import argparse
import json
import sys
import time
from collections import Counter
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=float, default=0.2, help="fraction of the simulate.json phase durations")
    ap.add_argument("--capacity", type=int, default=8, help="backlog that counts as a full buffer")
    ap.add_argument("--idle-ms", type=float, default=20.0)
    ap.add_argument("--min-k", type=int, default=2)
    ap.add_argument("--out", default="gpurun_out/serve_bursty.json")
    args = ap.parse_args()

    import torch

    from paper_2408_12526_b200 import PRESETS, StudentGroup, random_bert_group
    from paper_2408_12526_b200.serving import AdaptiveServer, generate_phases, synth_tokens

    cfg, K = PRESETS["base"]
    group = StudentGroup(random_bert_group(cfg, K, seed=0), max_tokens=512, max_seqs=1)
    phases = [(2000.0, 4000.0 * args.scale), (10000.0, 2500.0 * args.scale), (2000.0, 18000.0 * args.scale)]
    trace = generate_phases(phases, seed=0, max_len=512, bin_width=32)
    tokens = {r.id: synth_tokens(r, 0, cfg.vocab) for r in trace}
    cu_cache = {}

    def execute(req, k):
        ids = tokens[req.id]
        cu = cu_cache.setdefault(len(ids), np.array([0, len(ids)], np.int32))
        t0 = time.perf_counter()
        group.forward_host(ids, cu, k)
        return 1e3 * (time.perf_counter() - t0)

    for k in range(args.min_k, K + 1):  # a server captures its graphs ahead of time (every k it may pick)
        group.prepare_graphs(512, k)
    for r in trace[:50]:  # warm-up (not part of the trace replay)
        execute(r, K)
    torch.cuda.synchronize()
    out = {"trace": {"phases_rps_ms": phases, "requests": len(trace), "len_range": [1, 512]}}
    for name, kmin in [("adaptive", args.min_k), ("fixed_k8", K)]:
        srv = AdaptiveServer(execute, max_students=K, min_students=kmin, buffer_capacity=args.capacity,
                             idle_window_ms=args.idle_ms)
        t0 = time.perf_counter()
        m = srv.run(trace)
        wall = time.perf_counter() - t0
        ks = Counter(r.k for r in m.records)
        svc = [r.completion_ms - r.start_ms for r in m.records]
        out[name] = {
            "p50_ms": m.p50_ms, "p99_ms": m.p99_ms, "avg_ms": m.avg_ms, "completed": m.completed,
            "service_p50_ms": float(np.percentile(svc, 50)), "k_histogram": dict(sorted(ks.items())),
            "k_changes": len(m.k_timeline) - 1, "min_k_seen": min(ks), "replay_wall_s": wall,
        }
        print(name, json.dumps(out[name]), flush=True)
    Path(args.out).parent.mkdir(parents=True, exist_ok=True)
    Path(args.out).write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()

"""Bursty Poisson trace with adaptive student count on the real engine (BASELINE.json config 4).

The trace has the reference's phase shape and rates (pkg/configs/simulate.json: 2000 -> 10000 ->
2000 rps) built exactly as cli.py:191-202 builds it (serving.generate_phases), lengths from the
reference's 16-bin histogram scaled to L <= 512. serving.AdaptiveServer replays it with the
reference's event semantics (servesim.py:430-549) and the measured wall time of every launch
through StudentGroup.forward_host (one C call: H2D ids, forward, D2H logits) in place of the
analytic service_time (servesim.py:486). No batching wait, no padding. Servers compared:
  single   one request per launch (bucket CUDA graphs), adaptive k in [2, 8]
  batched  continuous batching: the queued backlog packed into one unpadded launch (cu_seqlens, up to
           64 requests / 8192 tokens) whenever the engine is free, adaptive k in [2, 8]
  fixed_k8 single, k pinned at 8

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
    ap.add_argument("--capacity", type=int, default=64, help="queued requests that count as a full buffer")
    ap.add_argument("--idle-ms", type=float, default=20.0)
    ap.add_argument("--min-k", type=int, default=2)
    ap.add_argument("--out", default="gpurun_out/serve_bursty.json")
    args = ap.parse_args()

    import torch

    from paper_2408_12526_b200 import PRESETS, StudentGroup, random_bert_group
    from paper_2408_12526_b200.serving import AdaptiveServer, generate_phases, synth_tokens

    cfg, K = PRESETS["base"]
    group = StudentGroup(random_bert_group(cfg, K, seed=0), max_tokens=8192, max_seqs=64)
    phases = [(2000.0, 4000.0 * args.scale), (10000.0, 2500.0 * args.scale), (2000.0, 18000.0 * args.scale)]
    trace = generate_phases(phases, seed=0, max_len=512, bin_width=32)
    tokens = {r.id: synth_tokens(r, 0, cfg.vocab) for r in trace}

    def execute(batch, k, active):
        ids = tokens[batch[0].id] if len(batch) == 1 else np.concatenate([tokens[r.id] for r in batch])
        cu = np.zeros(len(batch) + 1, np.int32)
        cu[1:] = np.cumsum([len(tokens[r.id]) for r in batch])
        t0 = time.perf_counter()
        group.forward_host(ids, cu, k)
        return 1e3 * (time.perf_counter() - t0)

    for k in range(args.min_k, K + 1):  # a server captures its graphs ahead of time (every k it may pick)
        group.prepare_graphs(512, k)
    for r in trace[:50]:  # warm-up (not part of the trace replay)
        execute([r], K, 1)
        execute(trace[:16], K, 1)
    torch.cuda.synchronize()
    out = {"trace": {"phases_rps_ms": phases, "requests": len(trace), "len_range": [1, 512],
                     "source": "pkg/configs/simulate.json phases (durations x scale), cli.py:191-202"}}
    servers = {
        "single": dict(min_students=args.min_k, max_batch_seqs=1),
        "batched": dict(min_students=args.min_k, max_batch_seqs=64, max_batch_tokens=8192),
        "fixed_k8": dict(min_students=K, max_batch_seqs=1),
    }
    for name, kw in servers.items():
        srv = AdaptiveServer(execute, max_students=K, buffer_capacity=args.capacity, idle_window_ms=args.idle_ms, **kw)
        t0 = time.perf_counter()
        m = srv.run(trace)
        wall = time.perf_counter() - t0
        ks = Counter(r.k for r in m.records)
        span = max(r.completion_ms for r in m.records) - min(r.arrival_ms for r in m.records)
        out[name] = {
            "p50_ms": m.p50_ms, "p99_ms": m.p99_ms, "avg_ms": m.avg_ms, "completed": m.completed,
            "req_per_s_per_gpu": 1000.0 * m.completed / span, "launches": len(srv.batches),
            "mean_batch": float(np.mean(srv.batches)), "max_batch": int(max(srv.batches)),
            "k_histogram": {int(a): int(b) for a, b in sorted(ks.items())}, "k_changes": len(m.k_timeline) - 1,
            "rejected_pushes": srv.rejected_pushes, "replay_wall_s": wall,
        }
        print(name, json.dumps(out[name]), flush=True)
    Path(args.out).parent.mkdir(parents=True, exist_ok=True)
    Path(args.out).write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()

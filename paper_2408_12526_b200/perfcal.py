"""Perf-model recalibration from measured B200 latency.

The reference sizes deployments with an analytic model (perfmodel.py:1-12)

    latency = D · t_unit · max(1, ceil(W·B·N²·M / (C·G))) + Q(B) + B·N/T + gather

whose single constant t_unit (per-layer unit time) is solved from one observed configuration
(PerfModel.calibrate, perfmodel.py:108-122): the 12-layer, width-768 baseline at B=8, N=128 served
with dynamic batching (baseline_reference, :153-160), observed at 11.6 ms on the paper's GPUs
(REFERENCE_OBSERVED_LATENCY_MS, :150). The stock `perf` and `simulate` commands read that
observation from their config's ``calibration`` block (cli.py:124-140, :346-356).

This module MEASURES the calibration configuration on the B200 engine (a 12-layer BERT-base
encoder, batch 8 × 128 tokens, CUDA events, L2 flushed) and returns a reference-compatible
``calibration`` block: observed_latency_ms = measured compute + the model's own wait / transfer /
gather terms, so the reference's calibrate() solves exactly t_unit = measured / (D · waves). It
also measures the model's student-parallel row (student_parallel_factors, :163-180) on the engine
and reports how far the recalibrated model's prediction is from the measurement.

The model arithmetic below restates perfmodel.py so the engine package does not import the
reference (it does not exist on deployment hosts); tests pin it against the reference.
"""
from __future__ import annotations

import argparse
import json
import math
from dataclasses import dataclass, replace

import numpy as np

# perfmodel.py:145-150
DEFAULT_CAPACITY = 1.5e7
DEFAULT_PCIE_TOKENS_PER_MS = 1000.0
DEFAULT_GATHER_MS = 0.2
DEFAULT_BATCH_TIMEOUT_MS = 10.0
REFERENCE_OBSERVED_LATENCY_MS = 11.6


@dataclass(frozen=True)
class Factors:
    """PerfFactors (perfmodel.py:29-52) with the dynamic-batch wait model inlined."""

    depth: int
    width: int
    batch: int
    seq_len: int
    parallel_models: int
    gpus: int
    capacity: float = DEFAULT_CAPACITY
    pcie_tokens_per_ms: float = DEFAULT_PCIE_TOKENS_PER_MS
    gather_ms: float = 0.0
    timeout_ms: float | None = None  # DynamicBatch.timeout_ms (None: no batching wait)
    arrival_rps: float | None = None

    def __post_init__(self):  # perfmodel.py:42-48
        if min(self.depth, self.width, self.batch, self.seq_len, self.parallel_models, self.gpus) < 1:
            raise ValueError("all counts must be >= 1")
        if self.capacity <= 0 or self.pcie_tokens_per_ms <= 0:
            raise ValueError("capacity and pcie_tokens_per_ms must be positive")
        if self.gather_ms < 0:
            raise ValueError("gather_ms must be nonnegative")


def waiting_time(f: Factors) -> float:
    """perfmodel.py:62-68."""
    if f.timeout_ms is None:
        return 0.0
    if f.arrival_rps is None or f.arrival_rps <= 0:
        raise ValueError("arrival_rps must be positive under dynamic batching")
    return min(f.timeout_ms, 1000.0 * (f.batch - 1) / (2.0 * f.arrival_rps))


def compute_waves(f: Factors) -> int:
    """perfmodel.py:71-74."""
    work = float(f.width) * f.batch * f.seq_len ** 2 * f.parallel_models
    return max(1, math.ceil(work / (f.capacity * f.gpus)))


def transfer_term(f: Factors) -> float:
    """perfmodel.py:89-91."""
    return f.batch * f.seq_len / f.pcie_tokens_per_ms


def fixed_terms(f: Factors) -> float:
    return waiting_time(f) + transfer_term(f) + f.gather_ms


def latency(f: Factors, t_unit: float) -> float:
    """perfmodel.py:93-99 (same summation order)."""
    return f.depth * t_unit * compute_waves(f) + waiting_time(f) + transfer_term(f) + f.gather_ms


def calibrate(reference: Factors, observed_latency_ms: float) -> float:
    """PerfModel.calibrate (perfmodel.py:108-122): t_unit with latency(reference) == observed."""
    residual = observed_latency_ms - fixed_terms(reference)
    if residual <= 0:
        raise ValueError(f"infeasible calibration: observed {observed_latency_ms} ms does not exceed "
                         f"the wait/transfer/gather floor {fixed_terms(reference):.3f} ms")
    return residual / (reference.depth * compute_waves(reference))


def baseline_reference(gpus: int = 4, arrival_rps: float = 2000.0) -> Factors:
    """perfmodel.py:153-160."""
    return Factors(depth=12, width=768, batch=8, seq_len=128, parallel_models=gpus, gpus=gpus,
                   timeout_ms=DEFAULT_BATCH_TIMEOUT_MS, arrival_rps=arrival_rps)


def student_parallel_factors(gpus: int = 4, students: int = 3, width_per_student: int = 256, depth: int = 2,
                             typical_len: int = 32, batch: int = 4) -> Factors:
    """perfmodel.py:163-180."""
    return Factors(depth=depth, width=width_per_student * students, batch=batch, seq_len=typical_len,
                   parallel_models=4 * gpus, gpus=gpus,
                   gather_ms=DEFAULT_GATHER_MS if students > 1 and gpus > 1 else 0.0)


def reference_factor_rows(gpus: int = 4, arrival_rps: float = 2000.0) -> list[tuple[str, Factors]]:
    """The six stock rows of the factor ledger (perfmodel.py:183-197)."""
    base = baseline_reference(gpus, arrival_rps)
    return [
        ("bert_base_12l", base),
        ("tinybert_4l", replace(base, depth=4, width=312)),
        ("dynabert_6l", replace(base, depth=6, width=192)),
        ("deebert_early_exit", replace(base, depth=7, width=768)),
        ("cocktail_bagging", replace(base, depth=12, width=768 + 312 + 192 + 768)),
        ("student_parallel_2l", student_parallel_factors(gpus)),
    ]


def throughput_per_gpu(f: Factors, latency_ms: float) -> float:
    """perfmodel.py:101-106."""
    if latency_ms <= 0:
        raise ValueError("latency must be positive")
    return 1000.0 * f.batch * f.parallel_models / (latency_ms * f.gpus)


# ---------------------------------------------------------------------------- measurement (GPU)
def measure_engine_ms(hidden: int, n_layers: int, n_heads: int, n_students: int, batch: int, seq_len: int,
                      reps: int = 30, warmup: int = 5, seed: int = 0) -> float:
    """Median device time (ms) of one engine forward: `n_students` BERT students of the given shape on
    `batch` sequences of `seq_len` tokens, CUDA events on the launching stream, L2 flushed before
    every rep (write + read of 2 x 256 MiB)."""
    import torch

    from .group import StudentGroup
    from .weights import BertConfig, random_bert_group

    cfg = BertConfig(hidden=hidden, n_layers=n_layers, n_heads=n_heads)
    w = random_bert_group(cfg, n_students, seed=seed)
    T = batch * seq_len
    grp = StudentGroup(w, max_tokens=T, max_seqs=batch)
    rng = np.random.default_rng(seed)
    ids = np.concatenate([np.r_[101, rng.integers(1000, cfg.vocab, size=seq_len - 1)] for _ in range(batch)])
    dev = grp.device
    ids_d = torch.tensor(ids, dtype=torch.int32, device=dev)
    cu_d = torch.arange(0, T + 1, seq_len, dtype=torch.int32, device=dev)
    logits = torch.empty((batch, cfg.n_classes), dtype=torch.float32, device=dev)
    fw = torch.empty(256 << 18, device=dev)
    fr = torch.ones(256 << 18, device=dev)
    run = lambda: grp.forward_packed_device(ids_d, cu_d, batch, T, seq_len, n_students, None, logits)  # noqa: E731
    for _ in range(warmup):
        run()
    torch.cuda.synchronize(dev)
    ts = []
    for _ in range(reps):
        fw.zero_()
        fr.sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run()
        e1.record()
        torch.cuda.synchronize(dev)
        ts.append(e0.elapsed_time(e1))
    grp.close()
    return float(np.median(ts))


def calibrate_b200(gpus: int = 4, arrival_rps: float = 2000.0, reps: int = 30) -> dict:
    """Measure the reference's calibration configuration and its student-parallel row on this GPU;
    return the recalibrated model and a drop-in ``calibration`` block for the reference's configs."""
    base = baseline_reference(gpus, arrival_rps)
    # one model per GPU (M = G): the per-GPU work is one 12-layer, width-768 encoder
    measured = measure_engine_ms(base.width, base.depth, 12, 1, base.batch, base.seq_len, reps=reps)
    observed = measured + fixed_terms(base)
    t_unit = calibrate(base, observed)
    sp = student_parallel_factors(gpus)
    # a student-parallel group: 3 students of width 256 (4 heads of 64), 2 layers, B=4, N=32
    sp_ms = measure_engine_ms(256, sp.depth, 4, 3, sp.batch, sp.seq_len, reps=reps)
    rows = {name: {"latency_ms": latency(f, t_unit), "throughput_per_gpu": throughput_per_gpu(f, latency(f, t_unit))}
            for name, f in reference_factor_rows(gpus, arrival_rps)}
    return {
        "factor_table": rows,
        "calibration": {"observed_latency_ms": observed, "gpus": gpus, "arrival_rps": arrival_rps},
        "t_unit_ms": t_unit,
        "reference_t_unit_ms": calibrate(base, REFERENCE_OBSERVED_LATENCY_MS),
        "measured": {"baseline_compute_ms": measured, "baseline_waves": compute_waves(base),
                     "fixed_terms_ms": fixed_terms(base)},
        "student_parallel": {
            "measured_compute_ms": sp_ms,
            "predicted_compute_ms": sp.depth * t_unit * compute_waves(sp),
            "predicted_latency_ms": latency(sp, t_unit),
            "measured_latency_ms": sp_ms + fixed_terms(sp),
        },
    }


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description="Recalibrate the reference's perf model from measured B200 latency")
    ap.add_argument("--gpus", type=int, default=4)
    ap.add_argument("--arrival-rps", type=float, default=2000.0)
    ap.add_argument("--reps", type=int, default=30)
    ap.add_argument("--out", default=None, help="write the result JSON here (else stdout)")
    a = ap.parse_args(argv)
    res = calibrate_b200(a.gpus, a.arrival_rps, a.reps)
    text = json.dumps(res, indent=1)
    if a.out:
        with open(a.out, "w", encoding="utf-8") as fh:
            fh.write(text + "\n")
    print(text)
    return 0


if __name__ == "__main__":
    raise SystemExit(main())

"""Serving-side pieces of the hot path: request stream, adaptive student count, request metric.

Restated from the reference's discrete-event simulator (it never runs a model) so the
real engine can replace its analytic ``service_time`` (servesim.py:287-307):

* ``generate_workload`` — Poisson arrivals with a 16-bin length histogram (servesim.py:57-98)
  and multi-phase bursts (cli.py:191-202); deterministic per seed (seeding.py:19-21).
* ``decide_controller_action`` — DROP_ONE / ADD_ONE / HOLD (servesim.py:317-342).
* ``nearest_rank_percentile`` — the p50/p99 definition of the metric (servesim.py:370-376).
* ``AdaptiveServer`` — the serving loop on the real engine: the simulator's event loop
  (servesim.py:430-549: arrivals, completions, 100 ms heartbeats; retries, controller tick and
  dispatch at every boundary) with the analytic service time replaced by the measured execution of
  a launch. Queued requests are packed into ONE unpadded launch (cu_seqlens) up to a token budget
  the moment an engine slot is free — no batching wait, no padding; ``max_batch_seqs=1`` is the
  single-request-in-flight server. k is snapshotted per launch (servesim.py:486).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .seeding import fork_seed, rng_for

DEFAULT_LENGTH_WEIGHTS = (1.0, 2.0, 3.0, 3.0, 2.0, 1.5, 1.0, 0.8, 0.6, 0.5, 0.4, 0.3, 0.25, 0.2, 0.15, 0.1)

DROP_ONE = "drop_one"
ADD_ONE = "add_one"
HOLD = "hold"


@dataclass(frozen=True)
class Request:
    id: int
    arrival_ms: float
    length_tokens: int


@dataclass(frozen=True)
class PoissonSpec:
    rps: float
    duration_ms: float
    length_weights: tuple[float, ...] | None = None


def generate_workload(spec: PoissonSpec, seed: int, max_len: int = 128, bin_width: int = 8) -> list[Request]:
    """Arrival-sorted Poisson requests (servesim.py:57-77): exponential gaps of mean 1000/rps ms,
    length bin drawn from the weight histogram, length uniform inside the bin."""
    if spec.rps <= 0:
        raise ValueError("rps must be positive")
    rng = rng_for(seed, "workload")
    weights = np.asarray(spec.length_weights or DEFAULT_LENGTH_WEIGHTS, dtype=np.float64)
    n_bins = len(weights)
    if n_bins * bin_width > max_len:
        raise ValueError("length_weights cover more than max_len tokens")
    probs = weights / weights.sum()
    out = []
    t = rng.exponential(1000.0 / spec.rps)
    rid = 0
    while t <= spec.duration_ms:
        b = int(rng.choice(n_bins, p=probs))
        length = int(rng.integers(b * bin_width + 1, (b + 1) * bin_width + 1))
        out.append(Request(rid, t, length))
        rid += 1
        t += rng.exponential(1000.0 / spec.rps)
    return out


def generate_phases(phases: list[tuple[float, float]], seed: int, max_len: int = 128, bin_width: int = 8,
                    length_weights=None) -> list[Request]:
    """Bursty trace: consecutive (rps, duration_ms) phases, each a Poisson segment seeded with
    fork_seed(seed, "workload-phase-i") and shifted to start where the previous phase ended;
    ids are renumbered in arrival order (cli.py:191-202)."""
    out: list[Request] = []
    offset = 0.0
    for i, (rps, dur) in enumerate(phases):
        seg = generate_workload(PoissonSpec(rps, dur, length_weights), fork_seed(seed, f"workload-phase-{i}"),
                                max_len, bin_width)
        for r in seg:
            out.append(Request(len(out), r.arrival_ms + offset, r.length_tokens))
        offset += dur
    return out


def decide_controller_action(k: int, min_students: int, max_students: int, any_buffer_full: bool,
                             all_buffers_idle_ms: float | None, idle_students: int, occupied_students: int,
                             idle_window_ms: float) -> str:
    """servesim.py:317-342: drop one student when a buffer has filled (and k > min); add one back
    after the idle window when idle capacity outweighs occupied capacity; otherwise hold."""
    if any_buffer_full and k > min_students:
        return DROP_ONE
    if (k < max_students and all_buffers_idle_ms is not None and all_buffers_idle_ms >= idle_window_ms
            and idle_students > occupied_students):
        return ADD_ONE
    return HOLD


def nearest_rank_percentile(values, pct: float) -> float:
    """The ceil(pct/100 * n)-th smallest value (servesim.py:370-376)."""
    values = list(values)
    if not values:
        raise ValueError("no values")
    ordered = sorted(values)
    rank = max(1, math.ceil(pct / 100.0 * len(ordered)))
    return ordered[rank - 1]


def synth_tokens(req: Request, seed: int, vocab: int) -> np.ndarray:
    """Token ids of a synthetic request: [CLS]=101 then U[1000, vocab)."""
    rng = rng_for(seed, f"tokens-{req.id}")
    ids = rng.integers(1000, vocab, size=req.length_tokens).astype(np.int32)
    ids[0] = 101
    return ids


@dataclass
class ServeRecord:
    request_id: int
    arrival_ms: float
    start_ms: float
    completion_ms: float
    k: int
    length_tokens: int

    @property
    def latency_ms(self) -> float:
        return self.completion_ms - self.arrival_ms


@dataclass
class ServeMetrics:
    p50_ms: float
    p99_ms: float
    avg_ms: float
    completed: int
    k_timeline: list[tuple[float, int]] = field(default_factory=list)
    records: list[ServeRecord] = field(default_factory=list, repr=False)


HEARTBEAT_MS = 100.0  # servesim.py:411


def group_count(group_size: int, gpus: int, replicas_per_gpu: int) -> int:
    """Replica groups a node hosts: floor(replicas x G / S), at least 1 (servesim.py:220-222)."""
    return max(1, (replicas_per_gpu * gpus) // group_size)


class AdaptiveServer:
    """Open-loop serving of an arrival trace on a real engine with the adaptive student count.

    ``execute(reqs, k, active) -> service_ms`` runs ONE launch on the engine: the requests ``reqs``
    packed unpadded (cu_seqlens), the first ``k`` students, while ``active`` launches are in flight
    (including this one), and returns its measured service time — it replaces the simulator's
    analytic service_time (servesim.py:486-487). Time is virtual: it advances by the measured
    service times, so the trace is replayed faithfully without sleeping.

    Event semantics follow Simulation (servesim.py:430-549): arrivals push into a bounded FIFO (a
    push into a full buffer is deferred to a retry queue, :519-523, :539-542); every event boundary
    first retries deferred pushes, then runs the controller (decide_controller_action with the
    real inputs: any buffer full, the time every buffer has been empty — None while a request is
    queued —, idle and occupied student slots, :497-517), then dispatches while a slot is free
    (:481-487), packing queued requests FIFO up to ``max_batch_seqs`` / ``max_batch_tokens``.
    Heartbeats every 100 ms let ADD_ONE fire during idle periods. ``slots(k)`` (default 1: one
    launch in flight per GPU) and ``capacity(k)`` (buffer capacity in requests) may depend on k like
    the reference's group_count (:220-222, :465-471).
    """

    def __init__(self, execute, max_students: int, min_students: int = 1, start_k: int | None = None,
                 buffer_capacity=8, idle_window_ms: float = 50.0, max_batch_seqs: int = 1,
                 max_batch_tokens: int = 1 << 30, slots=1):
        if not 1 <= min_students <= max_students:
            raise ValueError("need 1 <= min_students <= max_students")
        if max_batch_seqs < 1 or max_batch_tokens < 1:
            raise ValueError("batch limits must be >= 1")
        self.execute = execute
        self.max_students, self.min_students = max_students, min_students
        self.k = max_students if start_k is None else start_k
        if not min_students <= self.k <= max_students:
            raise ValueError("start_k outside [min_students, max_students]")
        self.capacity = buffer_capacity if callable(buffer_capacity) else (lambda k, c=buffer_capacity: c)
        self.slots = slots if callable(slots) else (lambda k, n=slots: n)
        self.idle_window_ms = idle_window_ms
        self.max_batch_seqs, self.max_batch_tokens = max_batch_seqs, max_batch_tokens
        self.actions: list[tuple[float, str]] = []
        self.batches: list[int] = []
        self.rejected_pushes = 0

    def run(self, requests: list[Request]) -> ServeMetrics:
        import heapq
        from collections import deque

        events: list = []
        seq = 0

        def push_event(t, kind, payload):
            nonlocal seq
            heapq.heappush(events, (t, seq, kind, payload))
            seq += 1

        for r in requests:
            push_event(r.arrival_ms, "arrival", r)
        horizon = max((r.arrival_ms for r in requests), default=0.0) + self.idle_window_ms + 5 * HEARTBEAT_MS
        t = 0.0
        while t <= horizon:
            push_event(t, "heartbeat", None)
            t += HEARTBEAT_MS
        queue: deque[Request] = deque()
        retry: deque[Request] = deque()
        busy = 0
        empty_since: float | None = 0.0
        timeline = [(0.0, self.k)]
        records: list[ServeRecord] = []

        def try_push(req) -> bool:
            if len(queue) >= self.capacity(self.k):
                return False
            queue.append(req)
            return True

        while events:
            now, _, kind, payload = heapq.heappop(events)
            if kind == "arrival":
                if retry or not try_push(payload):
                    self.rejected_pushes += 1
                    retry.append(payload)
            elif kind == "completion":
                start, k_b, batch = payload
                busy -= 1
                for req in batch:
                    records.append(ServeRecord(req.id, req.arrival_ms, start, now, k_b, req.length_tokens))
            # ---- event boundary (servesim.py:525-531)
            while retry and try_push(retry[0]):
                retry.popleft()
            idle_ms = (now - empty_since) if (not queue and empty_since is not None) else None
            slots = self.slots(self.k)
            action = decide_controller_action(self.k, self.min_students, self.max_students,
                                              len(queue) >= self.capacity(self.k), idle_ms,
                                              idle_students=max(0, slots - busy) * self.k,
                                              occupied_students=busy * self.k,
                                              idle_window_ms=self.idle_window_ms)
            if action == DROP_ONE:
                self.k -= 1
                timeline.append((now, self.k))
                self.actions.append((now, action))
            elif action == ADD_ONE:
                self.k += 1
                timeline.append((now, self.k))
                self.actions.append((now, action))
                if empty_since is not None:  # a fresh idle window must elapse before the next add
                    empty_since = now
            while busy < self.slots(self.k) and queue:
                batch = [queue.popleft()]
                tokens = batch[0].length_tokens
                while (queue and len(batch) < self.max_batch_seqs
                       and tokens + queue[0].length_tokens <= self.max_batch_tokens):
                    tokens += queue[0].length_tokens
                    batch.append(queue.popleft())
                busy += 1
                k_b = self.k  # snapshotted per dispatched launch (servesim.py:486)
                dt = float(self.execute(batch, k_b, busy))
                self.batches.append(len(batch))
                push_event(now + dt, "completion", (now, k_b, batch))
            if not queue:
                if empty_since is None:
                    empty_since = now
            else:
                empty_since = None
        records.sort(key=lambda r: (r.arrival_ms, r.request_id))
        lat = [r.latency_ms for r in records]
        return ServeMetrics(nearest_rank_percentile(lat, 50), nearest_rank_percentile(lat, 99),
                            float(np.mean(lat)), len(records), timeline, records)

"""Serving-side pieces of the hot path: request stream, adaptive student count, request metric.

Restated from the reference's discrete-event simulator (it never runs a model) so the
real engine can replace its analytic ``service_time`` (servesim.py:287-307):

* ``generate_workload`` — Poisson arrivals with a 16-bin length histogram (servesim.py:57-98)
  and multi-phase bursts (cli.py:191-202); deterministic per seed (seeding.py:19-21).
* ``decide_controller_action`` — DROP_ONE / ADD_ONE / HOLD (servesim.py:317-342).
* ``nearest_rank_percentile`` — the p50/p99 definition of the metric (servesim.py:370-376).
* ``AdaptiveServer`` — a live serving loop: requests are dispatched immediately on arrival
  (no batching wait, no padding), the active prefix k is snapshotted per request
  (servesim.py:486) and adapted by the controller rule from the observed backlog.
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


class AdaptiveServer:
    """Open-loop serving of an arrival trace on a real engine with the adaptive student count.

    ``execute(req, k) -> service_ms`` runs one request on the engine (batch-1, unpadded) and
    returns its measured service time; it replaces the simulator's analytic service_time
    (servesim.py:486-487). The server keeps one in-flight request per group (a FIFO of arrivals
    is the buffer); at each dispatch boundary the controller compares the backlog against
    ``buffer_capacity`` (DROP_ONE when full) and the time the queue has been empty (ADD_ONE
    after ``idle_window_ms``), exactly the rule of decide_controller_action. Time is virtual:
    it advances by the measured service times, so the trace is replayed faithfully without
    sleeping.
    """

    def __init__(self, execute, max_students: int, min_students: int = 1, start_k: int | None = None,
                 buffer_capacity: int = 8, idle_window_ms: float = 50.0):
        if not 1 <= min_students <= max_students:
            raise ValueError("need 1 <= min_students <= max_students")
        self.execute = execute
        self.max_students, self.min_students = max_students, min_students
        self.k = max_students if start_k is None else start_k
        if not min_students <= self.k <= max_students:
            raise ValueError("start_k outside [min_students, max_students]")
        self.capacity = buffer_capacity
        self.idle_window_ms = idle_window_ms

    def run(self, requests: list[Request]) -> ServeMetrics:
        now = 0.0
        queue: list[Request] = []
        i = 0
        idle_since: float | None = 0.0
        timeline = [(0.0, self.k)]
        records: list[ServeRecord] = []
        n = len(requests)
        while i < n or queue:
            while i < n and requests[i].arrival_ms <= now:
                queue.append(requests[i])
                i += 1
            if not queue:
                now = requests[i].arrival_ms
                continue
            # controller boundary (servesim.py:497-531): buffer full -> drop; long idle -> add
            idle_ms = None if idle_since is None else now - idle_since
            action = decide_controller_action(self.k, self.min_students, self.max_students,
                                              len(queue) >= self.capacity, idle_ms,
                                              idle_students=self.k, occupied_students=0,  # the group is idle here
                                              idle_window_ms=self.idle_window_ms)
            if action == DROP_ONE:
                self.k -= 1
                timeline.append((now, self.k))
            elif action == ADD_ONE:
                self.k += 1
                idle_since = now
                timeline.append((now, self.k))
            req = queue.pop(0)
            k_req = self.k  # snapshotted per dispatched request (servesim.py:486)
            service = float(self.execute(req, k_req))
            start = now
            now = now + service
            records.append(ServeRecord(req.id, req.arrival_ms, start, now, k_req, req.length_tokens))
            while i < n and requests[i].arrival_ms <= now:
                queue.append(requests[i])
                i += 1
            if queue:
                idle_since = None
            elif idle_since is None:
                idle_since = now
        lat = [r.latency_ms for r in records]
        return ServeMetrics(nearest_rank_percentile(lat, 50), nearest_rank_percentile(lat, 99),
                            float(np.mean(lat)), len(records), timeline, records)

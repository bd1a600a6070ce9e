"""Student parallelism across GPUs: placement, prefix-k per shard, and the single logit reduce.

Students are independent during inference (distill.py:175-177), so a K-student group shards into
K/n students per GPU with exactly ONE exchange per request: every rank computes the alpha-weighted
partial logits of its local students, z_g = W_c * sum_{m in g, m < k} alpha_m S_m(x) (no bias),
and one NCCL all-reduce sums them; the classifier bias is added exactly once (on the root's
partial) — exact by linearity of the identity classifier (distill.py:535).

Placement follows the reference's allocate_students (servesim.py:225-234) for one group (j = 0):
student i -> GPU i mod G. Round-robin keeps the load balanced when the adaptive controller drops
trailing students (prefix-k).
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def placement(n_students: int, world: int) -> list[list[int]]:
    """Global student indices held by each rank: i -> i mod world (servesim.py:231 with j = 0)."""
    if n_students < 1 or world < 1:
        raise ValueError("n_students and world must be >= 1")  # servesim.py:227-228
    return [[i for i in range(n_students) if i % world == r] for r in range(world)]


def local_prefix(k: int, students: list[int], total: int) -> int:
    """How many of this rank's students lie in the global prefix [0, k) (distill.py:171-173)."""
    if not 1 <= k <= total:
        raise ValueError(f"k={k} out of range 1..{total}")
    return sum(1 for i in students if i < k)


def reduce_partials(partial: torch.Tensor, group=None) -> torch.Tensor:
    """Sum per-rank partial logits in place (one all-reduce; NCCL on GPU, gloo in CPU tests)."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(partial, op=dist.ReduceOp.SUM, group=group)
    return partial


class ShardedStudentGroup:
    """This rank's shard of a K-student group (BERT kind), answering for the whole group."""

    def __init__(self, cfg, n_students: int, seed: int = 0, rank: int | None = None, world: int | None = None,
                 device: int | None = None, max_tokens: int = 4096, max_seqs: int = 256, weights=None,
                 process_group=None):
        from .group import StudentGroup
        from .weights import random_bert_group

        self.rank = dist.get_rank() if rank is None and dist.is_initialized() else (rank or 0)
        self.world = dist.get_world_size() if world is None and dist.is_initialized() else (world or 1)
        self.total = n_students
        self.students = placement(n_students, self.world)[self.rank]
        if not self.students:
            raise ValueError(f"rank {self.rank} holds no students (K={n_students} < world={self.world})")
        self.process_group = process_group
        if weights is None:
            weights = random_bert_group(cfg, n_students, seed=seed, students=self.students)
        elif weights.n_students != len(self.students):
            weights = weights.subset(self.students)
        dev = torch.cuda.current_device() if device is None else device
        self.local = StudentGroup(weights, device=dev, max_tokens=max_tokens, max_seqs=max_seqs,
                                  global_index=self.students)
        self.device = self.local.device
        self.n_classes = self.local.n_classes
        self._pinned_logits = None

    def local_k(self, k: int | None) -> int:
        return local_prefix(self.total if k is None else int(k), self.students, self.total)

    def forward_packed_device(self, ids, cu, n_seqs, n_tokens, max_len, k, logits, stream=None, graph=True):
        """Device buffers in, reduced logits (identical on every rank) out; no host sync.
        A single sequence replays this shard's 16-token bucket graph (one launch instead of ~15
        on every rank); a shard with no student in the prefix writes zero partials eagerly."""
        kl = self.local_k(k)
        if graph and n_seqs == 1 and kl >= 1:
            self.local.forward_graph_device(ids, cu, n_tokens, kl, logits, add_bias=(self.rank == 0), stream=stream)
        else:
            self.local.forward_packed_device(ids, cu, n_seqs, n_tokens, max_len, kl, None, logits,
                                             add_bias=(self.rank == 0), stream=stream)
        reduce_partials(logits[:n_seqs], self.process_group)
        return logits

    def _ensure_staging(self):
        if self._pinned_logits is None:  # staging allocated once (pinned: async copies, no per-call alloc)
            dev = self.device
            self._h_ids = torch.empty(self.local.max_tokens, dtype=torch.int32).pin_memory()
            self._h_cu = torch.empty(self.local.max_seqs + 1, dtype=torch.int32).pin_memory()
            self._d_ids = torch.empty(self.local.max_tokens, dtype=torch.int32, device=dev)
            self._d_cu = torch.empty(self.local.max_seqs + 1, dtype=torch.int32, device=dev)
            self._d_logits = torch.empty((self.local.max_seqs, self.n_classes), dtype=torch.float32, device=dev)
            self._pinned_logits = torch.empty((self.local.max_seqs, self.n_classes), dtype=torch.float32).pin_memory()

    def prepare_graphs(self, max_tokens: int | None = None, k: int | None = None) -> None:
        """Capture this shard's batch-1 bucket graphs of forward_host ahead of time (no collective)."""
        kl = self.local_k(k)
        if kl < 1:
            return
        self._ensure_staging()
        top = min(int(max_tokens or self.local.max_tokens), self.local.max_tokens, self.local.weights.cfg.max_pos)
        self._d_ids.fill_(1000)
        for t in range(16, top + 16, 16):
            t = min(t, top)
            self._d_cu[:2].copy_(torch.tensor([0, t], dtype=torch.int32))
            self.local.forward_graph_device(self._d_ids, self._d_cu, t, kl, self._d_logits, add_bias=(self.rank == 0))
        torch.cuda.synchronize(self.device)

    def forward_host(self, ids: np.ndarray, cu: np.ndarray, k: int | None = None) -> np.ndarray:
        """Public end-to-end call: host ids/cu_seqlens in, host logits out (every rank gets them)."""
        from .group import validate_packed

        cfg = self.local.weights.cfg
        ids = np.ascontiguousarray(ids, dtype=np.int32)
        cu = np.ascontiguousarray(cu, dtype=np.int32)
        max_len = validate_packed(ids, cu, cfg.vocab, cfg.max_pos)
        n, t = len(cu) - 1, len(ids)
        if n > self.local.max_seqs or t > self.local.max_tokens:
            raise ValueError(f"request ({n} seqs, {t} tokens) exceeds the group's capacity")
        self._ensure_staging()
        self._h_ids.numpy()[:t] = ids
        self._h_cu.numpy()[: n + 1] = cu
        self._d_ids[:t].copy_(self._h_ids[:t], non_blocking=True)
        self._d_cu[: n + 1].copy_(self._h_cu[: n + 1], non_blocking=True)
        self.forward_packed_device(self._d_ids, self._d_cu, n, t, max_len, k, self._d_logits)
        self._pinned_logits[:n].copy_(self._d_logits[:n], non_blocking=True)
        torch.cuda.current_stream(self.device).synchronize()
        return self._pinned_logits[:n].numpy().copy()

"""Student parallelism across GPUs: placement, prefix-k per shard, and the single logit reduce.

Students are independent during inference (distill.py:175-177), so a K-student group shards into
K/n students per GPU with exactly ONE exchange per request: every rank computes the alpha-weighted
partial logits of its local students, z_g = W_c * sum_{m in g, m < k} alpha_m S_m(x) (no bias),
and the partials are summed; the classifier bias is added exactly once (on the root's partial) —
exact by linearity of the identity classifier (distill.py:535). Two reduce paths:

* ``reduce="nccl"`` (baseline): one NCCL all-reduce of the partials; every rank gets the logits.
* ``reduce="p2p"``: the device-side mailbox reduce of sp_reduce.cu — every rank stores its
  partial into its slot of a mailbox on the root's GPU (CUDA-IPC mapping, NVLink) and raises a
  flag; the root's combine kernel sums the slots in fixed rank order. No collective, no host
  synchronisation; only the root returns the logits.

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


class LogitMailbox:
    """The root's mailbox of the device-side logit reduce (include/studentpar_b200.h sp_reduce_*).

    The root (rank 0) allocates it on its GPU; with torch.distributed initialised and world > 1 the
    other ranks map it through CUDA IPC (the 64-byte handle is broadcast over the process group).
    Shards built in ONE process (tests, one device) pass ``shared=`` the root's mailbox instead."""

    def __init__(self, world: int, rank: int, max_rows: int, n_classes: int, device: torch.device,
                 process_group=None, shared: "LogitMailbox | None" = None):
        import ctypes as C

        from . import _lib

        self._lib = _lib.load()
        self.world, self.rank, self.max_rows, self.n_classes = world, rank, max_rows, n_classes
        self._owner = False
        self._opened = False
        if shared is not None:
            self.ptr = shared.ptr
            return
        ptr = C.c_void_p()
        multi = world > 1 and dist.is_available() and dist.is_initialized()
        if rank == 0:
            _lib.check(self._lib.sp_mailbox_create(world, max_rows, n_classes, device.index, C.byref(ptr)))
            self._owner = True
            if multi:
                handle = (C.c_char * 64)()
                _lib.check(self._lib.sp_ipc_get_handle(ptr, handle))
                obj = [bytes(handle)]
                dist.broadcast_object_list(obj, src=0, group=process_group)
        elif multi:
            obj = [None]
            dist.broadcast_object_list(obj, src=0, group=process_group)
            handle = (C.c_char * 64).from_buffer_copy(obj[0])
            with torch.cuda.device(device):
                _lib.check(self._lib.sp_ipc_open_handle(handle, C.byref(ptr)))
            self._opened = True
        else:
            raise ValueError("a non-root shard needs the root's mailbox (shared=) or an initialised process group")
        self.ptr = ptr.value

    def publish(self, partial: torch.Tensor, n_rows: int, seq: int, stream) -> None:
        from . import _lib

        _lib.check(self._lib.sp_reduce_publish(self.ptr, partial.data_ptr(), self.rank, self.world, n_rows,
                                               self.max_rows, self.n_classes, seq, stream))

    def combine(self, n_rows: int, seq: int, out_ptr: int, flag_ptr: int | None, stream) -> None:
        from . import _lib

        _lib.check(self._lib.sp_reduce_combine(self.ptr, self.world, n_rows, self.max_rows, self.n_classes, seq,
                                               None, out_ptr, flag_ptr, stream))

    def close(self) -> None:
        if getattr(self, "_owner", False) and self.ptr:
            self._lib.sp_mailbox_destroy(self.ptr)
        elif getattr(self, "_opened", False) and self.ptr:
            self._lib.sp_ipc_close_handle(self.ptr)
        self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class ShardedStudentGroup:
    """This rank's shard of a K-student group (BERT kind), answering for the whole group."""

    def __init__(self, cfg, n_students: int, seed: int = 0, rank: int | None = None, world: int | None = None,
                 device: int | None = None, max_tokens: int = 4096, max_seqs: int = 256, weights=None,
                 process_group=None, reduce: str = "nccl", mailbox: LogitMailbox | None = None):
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
        if reduce not in ("nccl", "p2p"):
            raise ValueError(f"unknown reduce {reduce!r} (nccl | p2p)")
        self.reduce = reduce
        self.mailbox = None
        self._seq = 0
        if reduce == "p2p":
            self.mailbox = LogitMailbox(self.world, self.rank, max_seqs, self.n_classes, self.device,
                                        process_group=process_group, shared=mailbox)
            self._d_partial = torch.zeros((max_seqs, self.n_classes), dtype=torch.float32, device=self.device)

    def local_k(self, k: int | None) -> int:
        return local_prefix(self.total if k is None else int(k), self.students, self.total)

    def forward_packed_device(self, ids, cu, n_seqs, n_tokens, max_len, k, logits, stream=None, graph=True,
                              out_flag_ptr: int | None = None):
        """Device buffers in, reduced logits out; no host sync. A single sequence replays this
        shard's 16-token bucket graph (one launch instead of ~15 on every rank); a shard with no
        student in the prefix writes zero partials eagerly. NCCL: every rank's ``logits`` receive the
        sum. P2P: only the root's ``logits`` do (other ranks publish their partial and return);
        shards of one process must be called non-root first (the root's combine waits for them)."""
        kl = self.local_k(k)
        part = logits if self.reduce == "nccl" else self._d_partial
        if graph and n_seqs == 1 and kl >= 1:
            self.local.forward_graph_device(ids, cu, n_tokens, kl, part, add_bias=(self.rank == 0), stream=stream)
        else:
            self.local.forward_packed_device(ids, cu, n_seqs, n_tokens, max_len, kl, None, part,
                                             add_bias=(self.rank == 0), stream=stream)
        if self.reduce == "nccl":
            reduce_partials(logits[:n_seqs], self.process_group)
            return logits
        from .group import _stream_handle

        st = _stream_handle(stream, self.device)
        self._seq += 1
        self.mailbox.publish(self._d_partial, n_seqs, self._seq, st)
        if self.rank == 0:
            self.mailbox.combine(n_seqs, self._seq, logits.data_ptr(), out_flag_ptr, st)
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
            # p2p reduce: the root's combine writes logits + sequence flag straight into pinned memory
            self._h_out = torch.zeros((self.local.max_seqs, self.n_classes), dtype=torch.float32).pin_memory()
            self._h_flag = torch.zeros(16, dtype=torch.int32).pin_memory()
            self._staged = None

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

    def forward_host(self, ids: np.ndarray, cu: np.ndarray, k: int | None = None) -> np.ndarray | None:
        """Public end-to-end call: host ids/cu_seqlens in, host logits out. NCCL: every rank gets
        them (pinned D2H + stream sync). P2P: the root's combine writes the logits into mapped
        pinned memory and then the request's sequence number into a mapped flag the root polls (no
        stream synchronize); the other ranks enqueue their shard and publish, and return None."""
        from .group import validate_packed

        cfg = self.local.weights.cfg
        ids = np.ascontiguousarray(ids, dtype=np.int32)
        cu = np.ascontiguousarray(cu, dtype=np.int32)
        max_len = validate_packed(ids, cu, cfg.vocab, cfg.max_pos)
        n, t = len(cu) - 1, len(ids)
        if n > self.local.max_seqs or t > self.local.max_tokens:
            raise ValueError(f"request ({n} seqs, {t} tokens) exceeds the group's capacity")
        self._ensure_staging()
        if self._staged is not None:  # the previous request's H2D copies have read the pinned staging
            self._staged.synchronize()
        self._h_ids.numpy()[:t] = ids
        self._h_cu.numpy()[: n + 1] = cu
        self._d_ids[:t].copy_(self._h_ids[:t], non_blocking=True)
        self._d_cu[: n + 1].copy_(self._h_cu[: n + 1], non_blocking=True)
        self._staged = torch.cuda.Event()
        self._staged.record()
        if self.reduce == "p2p":
            flag = self._h_flag.numpy() if self.rank == 0 else None
            self.forward_packed_device(self._d_ids, self._d_cu, n, t, max_len, k, self._h_out,
                                       out_flag_ptr=self._h_flag.data_ptr() if self.rank == 0 else None)
            if self.rank != 0:
                return None
            seq = self._seq
            spins = 0
            while int(flag[0]) != (seq & 0x7FFFFFFF):
                spins += 1
                if spins % 4096 == 0:  # surface a failed launch instead of spinning forever
                    torch.cuda.current_stream(self.device).query()
            return self._h_out[:n].numpy().copy()
        self.forward_packed_device(self._d_ids, self._d_cu, n, t, max_len, k, self._d_logits)
        self._pinned_logits[:n].copy_(self._d_logits[:n], non_blocking=True)
        torch.cuda.current_stream(self.device).synchronize()
        return self._pinned_logits[:n].numpy().copy()

"""StudentGroup — the reference's ``EnsembleState`` API (distill.py:139-178) backed by the B200 engine.

    group = StudentGroup.from_ensemble(state)           # reference EnsembleState (dense StudentModel)
    group = StudentGroup.from_checkpoint("ensemble.json")
    group = StudentGroup(random_bert_group(cfg, 8))      # BERT-kind students
    rep = group.rep(x, k)          # EnsembleState.rep (distill.py:169-178)
    z   = group.logits(x, k)       # classifier.forward(rep) (distill.py:512)
    y   = group.predict(x, k)      # argmax (distill.py:513)

Inputs follow the reference conventions: the dense kind takes float rows ``x`` [n, d_in] (a 1-D
``x`` is one sample and the result is squeezed, nnkernel.py:67-70, :76); the BERT kind takes token
sequences — a list of int arrays, one 1-D int array (one sequence, squeezed), or a packed
``(ids, cu_seqlens)`` pair. ``k`` selects the prefix of the first k students (adaptive student
count); out-of-range k raises ValueError exactly like distill.py:171-173.

Weights are packed to the device ONCE (a snapshot, SURVEY §8b "Ownership"); the engine is
stateless per call and re-entrant per CUDA stream. There is no CPU fallback: without the CUDA
library or a GPU every call raises.
"""
from __future__ import annotations

import ctypes as C
from typing import Sequence

import numpy as np
import torch

from . import _lib
from .weights import BertGroupWeights, DenseGroupWeights, dense_group_from_ensemble


_TORCH_OPS = None


def torch_ops():
    """torch.ops.studentpar — the thin PyTorch C++ extension over the C ABI (csrc/sp_torch.cpp), or
    None if its library was not built (the ctypes binding of the same entry points is used then)."""
    global _TORCH_OPS
    if _TORCH_OPS is None:
        try:
            torch.ops.load_library(str(_lib.TORCH_LIB_PATH))
            _TORCH_OPS = torch.ops.studentpar
        except (OSError, RuntimeError):
            _TORCH_OPS = False
    return _TORCH_OPS or None


def _dev_tensor(a: np.ndarray, device: torch.device) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a)).to(device)


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def _stream_handle(stream: torch.cuda.Stream | None, device: torch.device) -> int:
    if stream is not None:
        return stream.cuda_stream
    if _raw_stream is not None:  # ~10x cheaper than building a torch.cuda.Stream object
        return _raw_stream(device.index if isinstance(device, torch.device) and device.index is not None
                           else torch.cuda.current_device())
    return torch.cuda.current_stream(device).cuda_stream


def pack_sequences(x) -> tuple[np.ndarray, np.ndarray, bool]:
    """Token input -> (ids int32 [T], cu_seqlens int32 [B+1], squeeze)."""
    if isinstance(x, tuple) and len(x) == 2:
        ids = np.ascontiguousarray(np.asarray(x[0]), dtype=np.int32)
        cu = np.ascontiguousarray(np.asarray(x[1]), dtype=np.int32)
        return ids, cu, False
    if isinstance(x, np.ndarray) and x.ndim == 1 and np.issubdtype(x.dtype, np.integer):
        seqs, squeeze = [x], True
    else:
        seqs, squeeze = list(x), False
    if not seqs:
        raise ValueError("no sequences")
    lens = [len(s) for s in seqs]
    cu = np.zeros(len(seqs) + 1, np.int32)
    cu[1:] = np.cumsum(lens)
    ids = np.ascontiguousarray(np.concatenate([np.asarray(s, dtype=np.int64) for s in seqs]).astype(np.int32))
    return ids, cu, squeeze


def validate_packed(ids: np.ndarray, cu: np.ndarray, vocab: int, max_pos: int) -> int:
    """Reference-style input validation (ValueError, never silent padding). Returns max length."""
    if cu.ndim != 1 or len(cu) < 2 or cu[0] != 0:
        raise ValueError("cu_seqlens must start at 0 and describe at least one sequence")
    lens = np.diff(cu.astype(np.int64))
    if (lens < 1).any():
        raise ValueError("every sequence needs at least one token (its CLS)")
    if lens.max() > max_pos:
        raise ValueError(f"sequence of {lens.max()} tokens exceeds max_pos {max_pos}")
    if cu[-1] != len(ids):
        raise ValueError(f"cu_seqlens[-1]={cu[-1]} != number of ids {len(ids)}")
    if len(ids) and (ids.min() < 0 or ids.max() >= vocab):
        raise ValueError("token id outside vocab")
    return int(lens.max())


class StudentGroup:
    """A boosting group of K students on one device (or the local shard of a multi-GPU group)."""

    def __init__(self, weights: BertGroupWeights | DenseGroupWeights, device: int | str | torch.device = 0,
                 max_tokens: int = 4096, max_seqs: int = 256, global_index: Sequence[int] | None = None):
        if not torch.cuda.is_available():
            raise RuntimeError("StudentGroup needs a CUDA device (the engine has no CPU fallback)")
        self._lib = _lib.load()
        self.weights = weights
        self.kind = weights.kind
        self.device = torch.device("cuda", device) if isinstance(device, int) else torch.device(device)
        if self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        K = weights.n_students
        # global student indices of the local students (prefix-k is over global indices)
        self.global_index = np.arange(K) if global_index is None else np.asarray(global_index, dtype=np.int64)
        if len(self.global_index) != K:
            raise ValueError("global_index must list one index per local student")
        self.multipliers = [float(a) for a in weights.alpha]
        self.max_tokens, self.max_seqs = int(max_tokens), int(max_seqs)
        self._tensors: dict[str, torch.Tensor] = {}
        cfg = _lib.SpConfig()
        cfg.n_students = K
        cfg.max_tokens = self.max_tokens
        cfg.max_seqs = self.max_seqs
        dev = self.device
        with torch.cuda.device(dev):
            if isinstance(weights, BertGroupWeights):
                c = weights.cfg
                cfg.kind = _lib.SP_KIND_BERT
                cfg.hidden, cfg.n_layers, cfg.n_heads, cfg.ffn = c.hidden, c.n_layers, c.n_heads, c.ffn
                cfg.vocab, cfg.max_pos, cfg.n_classes, cfg.ln_eps = c.vocab, c.max_pos, c.n_classes, c.ln_eps
                names = ["word_emb", "pos_emb", "type_emb", "emb_ln_gamma", "emb_ln_beta", "w_qkv", "b_qkv", "w_o",
                         "b_o", "ln1_gamma", "ln1_beta", "w_ffn1", "b_ffn1", "w_ffn2", "b_ffn2", "ln2_gamma",
                         "ln2_beta", "w_pool", "b_pool"]
                self.hidden, self.n_classes = c.hidden, c.n_classes
            elif isinstance(weights, DenseGroupWeights):
                cfg.kind = _lib.SP_KIND_DENSE
                cfg.hidden, cfg.n_layers, cfg.d_in = weights.hidden_padded, weights.depth, weights.d_in_padded
                cfg.n_classes = weights.n_classes
                names = ["w_in", "b_in", "w_layers", "b_layers"]
                if weights.exact_weights:
                    names += ["w_in_lo", "w_layers_lo"]
                self.hidden, self.n_classes = weights.hidden_padded, weights.n_classes
            else:
                raise TypeError(f"unsupported weights {type(weights).__name__}")
            for name in names + ["alpha", "w_cls", "b_cls"]:
                self._tensors[name] = _dev_tensor(getattr(weights, name), dev)
            torch.cuda.synchronize(dev)
            wst = _lib.SpWeights()
            for name, t in self._tensors.items():
                setattr(wst, name, t.data_ptr())
            handle = C.c_void_p()
            _lib.check(self._lib.sp_group_create(C.byref(cfg), C.byref(wst), dev.index, C.byref(handle)))
        self._handle = handle
        self._cfg = cfg

    # ------------------------------------------------------------------ construction helpers
    @classmethod
    def from_ensemble(cls, state, **kw) -> "StudentGroup":
        """Snapshot a reference ``EnsembleState`` (dense ``StudentModel`` students)."""
        return cls(dense_group_from_ensemble(state), **kw)

    @classmethod
    def from_checkpoint(cls, path, **kw) -> "StudentGroup":
        """Load an ``ensemble-checkpoint-v1`` file (distill.py:586-612)."""
        from .checkpoint import load_ensemble_weights

        return cls(load_ensemble_weights(path), **kw)

    def close(self) -> None:
        if getattr(self, "_handle", None):
            self._lib.sp_group_destroy(self._handle)
            self._handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __len__(self) -> int:
        return len(self.multipliers)

    @property
    def n_students(self) -> int:
        return len(self.multipliers)

    @property
    def last_launches(self) -> int:
        return int(self._lib.sp_group_last_launches(self._handle))

    def prepare_graphs(self, max_tokens: int | None = None, k: int | None = None, add_bias: bool = True) -> None:
        """Capture the batch-1 CUDA graphs of forward_host ahead of time (one per 16-token bucket)."""
        if self.kind != "bert":
            raise ValueError("graphs serve BERT-kind groups")
        kl = self.local_k(k)
        _lib.check(self._lib.sp_group_prepare_graphs(self._handle, int(max_tokens or self.max_tokens), kl,
                                                     int(add_bias)))

    def set_profiling(self, enable: bool) -> None:
        _lib.check(self._lib.sp_group_set_profiling(self._handle, int(enable)))

    def profile_records(self) -> list[dict]:
        """Per-launch device time / algorithmic bytes / flops of the last forward (profiling on)."""
        buf = (_lib.SpLaunchRecord * 256)()
        n = self._lib.sp_group_profile_read(self._handle, buf, 256)
        if n < 0:
            _lib.check(-n)
        return [dict(kind=_lib.LAUNCH_KINDS.get(r.kind, str(r.kind)), ms=float(r.ms), bytes=float(r.bytes),
                     flops=float(r.flops)) for r in buf[: min(n, 256)]]

    # ------------------------------------------------------------------ k handling
    def local_k(self, k: int | None, total: int | None = None) -> int:
        """Map the reference's global prefix k (distill.py:171-173) to the number of local students."""
        key = (k, total)
        cache = self.__dict__.setdefault("_local_k_cache", {})
        if key in cache:
            return cache[key]
        cache[key] = n = self._local_k(k, total)
        return n

    def _local_k(self, k: int | None, total: int | None) -> int:
        total = self.n_students if total is None else total
        k = total if k is None else int(k)
        if not 1 <= k <= total:
            raise ValueError(f"k={k} out of range 1..{total}")
        n = int(np.sum(self.global_index < k))
        if not np.all(self.global_index[:n] < k):
            raise ValueError("local students must be ordered by global index")
        return n

    # ------------------------------------------------------------------ device-level forward
    def forward_packed_device(self, ids: torch.Tensor, cu: torch.Tensor, n_seqs: int, n_tokens: int, max_len: int,
                              k_local: int, rep: torch.Tensor | None, logits: torch.Tensor, add_bias: bool = True,
                              stream: torch.cuda.Stream | None = None) -> None:
        """BERT kind on device buffers (no host sync). ``logits`` f32 [n_seqs, C] is written."""
        ops = torch_ops()
        if ops is not None and rep is None and stream is None:  # torch's current stream, checked tensors
            ops.group_forward(self._handle.value, ids, cu, n_seqs, n_tokens, max_len, k_local, logits, add_bias)
            return
        _lib.check(self._lib.sp_group_forward(self._handle, ids.data_ptr(), cu.data_ptr(), n_seqs, n_tokens, max_len,
                                              k_local, _ptr(rep), logits.data_ptr(), int(add_bias),
                                              _stream_handle(stream, self.device)))

    def forward_graph_device(self, ids: torch.Tensor, cu: torch.Tensor, n_tokens: int, k_local: int,
                             logits: torch.Tensor, add_bias: bool = True,
                             stream: torch.cuda.Stream | None = None) -> None:
        """One sequence on device buffers, replayed as its 16-token bucket's CUDA graph (no host sync)."""
        ops = torch_ops()
        if ops is not None and stream is None:
            ops.group_forward_graph(self._handle.value, ids, cu, n_tokens, k_local, logits, add_bias)
            return
        _lib.check(self._lib.sp_group_forward_graph(self._handle, ids.data_ptr(), cu.data_ptr(), n_tokens, k_local,
                                                    logits.data_ptr(), int(add_bias),
                                                    _stream_handle(stream, self.device)))

    def forward_dense_device(self, x16: torch.Tensor, n_rows: int, k_local: int, rep: torch.Tensor | None,
                             logits: torch.Tensor, add_bias: bool = True,
                             stream: torch.cuda.Stream | None = None, x16_lo: torch.Tensor | None = None) -> None:
        """Dense kind on device buffers: x16 fp16 [n_rows, d_in] (+ optional x16_lo, the fp16 residual of
        a wider input, read as a second operand term)."""
        _lib.check(self._lib.sp_group_forward_dense(self._handle, x16.data_ptr(), _ptr(x16_lo), n_rows, k_local,
                                                    _ptr(rep), logits.data_ptr(), int(add_bias),
                                                    _stream_handle(stream, self.device)))

    # ------------------------------------------------------------------ reference-facing API
    def _run(self, x, k, add_bias=True, want_rep=True, k_local=None, evaluate=False):
        dev = self.device
        if self.kind == "dense":
            w: DenseGroupWeights = self.weights
            xa = np.asarray(x, dtype=np.float64)
            squeeze = xa.ndim == 1
            if squeeze:
                xa = xa[None, :]
            if xa.ndim != 2 or xa.shape[1] != w.d_in:
                raise ValueError(f"input width {xa.shape} does not match layer in_dim {w.d_in}")  # nnkernel.py:71-72
            n = xa.shape[0]
            if n > self.max_tokens:
                raise ValueError(f"{n} rows exceed the group's capacity {self.max_tokens}")
            # the float64 input as an fp16 (hi, lo) pair: both operand terms of input_proj
            xp = np.zeros((2, n, w.d_in_padded), np.float16)
            xp[0, :, : w.d_in] = xa
            xp[1, :, : w.d_in] = xa - xp[0, :, : w.d_in].astype(np.float64)
            kl = self.local_k(k) if k_local is None else k_local
            with torch.cuda.device(dev):
                x16 = _dev_tensor(xp, dev)
                rep = torch.empty((n, self.hidden), dtype=torch.float32, device=dev) if want_rep else None
                if evaluate:
                    finals, prefix = self._eval_buffers(kl, n)
                    _lib.check(self._lib.sp_group_forward_dense_eval(self._handle, x16[0].data_ptr(),
                                                                     x16[1].data_ptr(), n, kl, finals.data_ptr(),
                                                                     prefix.data_ptr(), _stream_handle(None, dev)))
                    return finals[:, :, : w.rep_dim], prefix, squeeze, w.rep_dim
                logits = torch.empty((n, self.n_classes), dtype=torch.float32, device=dev)
                self.forward_dense_device(x16[0], n, kl, rep, logits, add_bias, x16_lo=x16[1])
            width = w.rep_dim
        else:
            ids, cu, squeeze = pack_sequences(x)
            cfg = self.weights.cfg
            max_len = validate_packed(ids, cu, cfg.vocab, cfg.max_pos)
            n = len(cu) - 1
            if n > self.max_seqs or len(ids) > self.max_tokens:
                raise ValueError(f"request ({n} seqs, {len(ids)} tokens) exceeds the group's capacity")
            kl = self.local_k(k) if k_local is None else k_local
            with torch.cuda.device(dev):
                ids_d = _dev_tensor(ids, dev)
                cu_d = _dev_tensor(cu, dev)
                rep = torch.empty((n, self.hidden), dtype=torch.float32, device=dev) if want_rep else None
                if evaluate:
                    finals, prefix = self._eval_buffers(kl, n)
                    _lib.check(self._lib.sp_group_forward_eval(self._handle, ids_d.data_ptr(), cu_d.data_ptr(), n,
                                                               len(ids), max_len, kl, finals.data_ptr(),
                                                               prefix.data_ptr(), _stream_handle(None, dev)))
                    return finals, prefix, squeeze, self.hidden
                logits = torch.empty((n, self.n_classes), dtype=torch.float32, device=dev)
                self.forward_packed_device(ids_d, cu_d, n, len(ids), max_len, kl, rep, logits, add_bias)
            width = self.hidden
        return rep, logits, squeeze, width

    def _eval_buffers(self, kl: int, n: int):
        if not np.array_equal(self.global_index, np.arange(self.n_students)):
            raise ValueError("training-side evaluation needs the whole group on one device (not a shard)")
        finals = torch.empty((kl, n, self.hidden), dtype=torch.float32, device=self.device)
        prefix = torch.empty((kl, n, self.n_classes), dtype=torch.float32, device=self.device)
        return finals, prefix

    def finals_and_prefix_logits(self, x, k: int | None = None) -> tuple[np.ndarray, np.ndarray]:
        """One GPU forward for training-side evaluation — the forward half of
        accumulate_prefix_gradients (distill.py:483-494): every student's final representation
        ``finals[m]`` = S_m(x) ([k, n, width], distill.py:483-486) and the logits of every prefix
        ``prefix[j-1]`` = classifier(sum_{m<j} alpha_m S_m(x)) ([k, n, C], :489-492), float64 copies.
        A 1-D (single-sample) input drops the sample axis, as rep() does (nnkernel.py:67-70)."""
        finals, prefix, squeeze, _ = self._run(x, k, evaluate=True)
        f = finals.double().cpu().numpy()
        z = prefix.double().cpu().numpy()
        return (f[:, 0], z[:, 0]) if squeeze else (f, z)

    def rep(self, x, k: int | None = None) -> np.ndarray:
        """Prefix-ensemble representation of the first k students (distill.py:169-178), float64."""
        rep, _, squeeze, width = self._run(x, k)
        out = rep[:, :width].double().cpu().numpy()
        return out[0] if squeeze else out

    def logits(self, x, k: int | None = None) -> np.ndarray:
        """classifier.forward(rep(x, k)) (distill.py:512), float64 copy of the fp32 logits."""
        _, logits, squeeze, _ = self._run(x, k, want_rep=False)
        out = logits.double().cpu().numpy()
        return out[0] if squeeze else out

    def predict(self, x, k: int | None = None) -> np.ndarray:
        """argmax of the logits (distill.py:513)."""
        z = np.atleast_2d(self.logits(x, k))
        return np.argmax(z, axis=1)

    def accuracy(self, x, labels, k: int) -> float:
        """prefix_accuracy (distill.py:508-513) on the engine."""
        return float(np.mean(self.predict(x, k) == np.asarray(labels)))

    def forward_host(self, ids: np.ndarray, cu: np.ndarray, k: int | None = None, add_bias: bool = True,
                     out: np.ndarray | None = None, stream: torch.cuda.Stream | None = None) -> np.ndarray:
        """End-to-end call with HOST buffers (ids in, logits out; the serving seam servesim.py:486).
        One C call: H2D of ids/cu_seqlens, the whole group forward, logits back on the host
        (batch-1: bucket-graph replay, logits via mapped pinned memory; else D2H + stream sync)."""
        if self.kind != "bert":
            raise ValueError("forward_host serves BERT-kind groups")
        ids = np.ascontiguousarray(ids, dtype=np.int32)
        cu = np.ascontiguousarray(cu, dtype=np.int32)
        n = len(cu) - 1
        if n < 1:
            raise ValueError("cu_seqlens must describe at least one sequence")
        if out is None:
            out = np.empty((n, self.n_classes), np.float32)
        elif (out.dtype != np.float32 or not out.flags.c_contiguous or out.ndim != 2
              or out.shape[0] < n or out.shape[1] != self.n_classes):
            raise ValueError(f"out must be a C-contiguous float32 array of shape (>= {n}, {self.n_classes})")
        kl = self.local_k(k)
        # host buffers: the direct C call (torch's current stream via the raw-stream getter) is 1.3 us
        # cheaper per request than wrapping three numpy arrays as tensors for the torch op
        # (tools/wrap_probe.py); torch.ops.studentpar.group_forward_host is the same entry point
        _lib.check(self._lib.sp_group_forward_host(self._handle, ids.ctypes.data, cu.ctypes.data, n, len(ids), kl,
                                                   out.ctypes.data, int(add_bias),
                                                   _stream_handle(stream, self.device)))
        return out

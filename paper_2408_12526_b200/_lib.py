"""ctypes binding of include/studentpar_b200.h (the engine's C ABI).

This is the binding a reference maintainer would add. There is no fallback:
if the library is missing or fails to load, every engine call raises.
"""
from __future__ import annotations

import ctypes as C
import threading
from pathlib import Path

from .build import LIB_PATH, TORCH_LIB_PATH

SP_OK, SP_EINVAL, SP_ECUDA, SP_ENOMEM = 0, 1, 2, 3
SP_KIND_DENSE, SP_KIND_BERT = 0, 1
ABI_VERSION = 3


class SpConfig(C.Structure):
    _fields_ = [
        ("kind", C.c_int32),
        ("n_students", C.c_int32),
        ("hidden", C.c_int32),
        ("n_layers", C.c_int32),
        ("n_heads", C.c_int32),
        ("ffn", C.c_int32),
        ("d_in", C.c_int32),
        ("vocab", C.c_int32),
        ("max_pos", C.c_int32),
        ("n_classes", C.c_int32),
        ("max_tokens", C.c_int32),
        ("max_seqs", C.c_int32),
        ("ln_eps", C.c_float),
    ]


_WEIGHT_FIELDS = [
    "word_emb", "pos_emb", "type_emb", "emb_ln_gamma", "emb_ln_beta",
    "w_qkv", "b_qkv", "w_o", "b_o", "ln1_gamma", "ln1_beta",
    "w_ffn1", "b_ffn1", "w_ffn2", "b_ffn2", "ln2_gamma", "ln2_beta",
    "w_pool", "b_pool",
    "w_in", "b_in", "w_layers", "b_layers",
    "alpha", "w_cls", "b_cls",
    "w_in_lo", "w_layers_lo",  # ABI v3: dense weight lo terms (optional)
]


class SpLaunchRecord(C.Structure):
    _fields_ = [("kind", C.c_int32), ("ms", C.c_float), ("bytes", C.c_double), ("flops", C.c_double)]


LAUNCH_KINDS = {1: "embed_ln", 2: "gemm_qkv", 3: "attention", 4: "gemm_o", 5: "reduce_ln", 6: "gemm_ffn1",
                7: "gemm_ffn2", 8: "gemm_pool", 9: "head", 10: "gemm_dense"}
GEMM_KINDS = {2, 4, 6, 7, 8, 10}


class SpWeights(C.Structure):
    _fields_ = [(name, C.c_void_p) for name in _WEIGHT_FIELDS]


# name -> (restype, argtypes); every symbol include/studentpar_b200.h declares
SIGNATURES: dict[str, tuple] = {
    "sp_abi_version": (C.c_int, []),
    "sp_last_error": (C.c_char_p, []),
    "sp_group_create": (C.c_int, [C.POINTER(SpConfig), C.POINTER(SpWeights), C.c_int, C.POINTER(C.c_void_p)]),
    "sp_group_destroy": (C.c_int, [C.c_void_p]),
    "sp_group_forward": (
        C.c_int,
        [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
         C.c_int32, C.c_void_p],
    ),
    "sp_group_forward_dense": (
        C.c_int,
        [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p],
    ),
    "sp_group_forward_eval": (
        C.c_int,
        [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
         C.c_void_p],
    ),
    "sp_group_forward_dense_eval": (
        C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p]
    ),
    "sp_group_forward_host": (
        C.c_int,
        [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_int32, C.c_void_p],
    ),
    "sp_group_last_launches": (C.c_int, [C.c_void_p]),
    "sp_group_prepare_graphs": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32]),
    "sp_group_forward_graph": (
        C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_int32, C.c_void_p],
    ),
    "sp_group_set_profiling": (C.c_int, [C.c_void_p, C.c_int]),
    "sp_group_profile_read": (C.c_int, [C.c_void_p, C.POINTER(SpLaunchRecord), C.c_int]),
    "sp_op_gemm": (
        C.c_int,
        [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
         C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p],
    ),
    "sp_debug_set_gemm_trace": (C.c_int, [C.c_void_p]),
    "sp_debug_set_attn_trace": (C.c_int, [C.c_void_p]),
    "sp_debug_gemm_trace_launches": (C.c_int, [C.c_void_p, C.c_int32]),
    "sp_reduce_mailbox_bytes": (C.c_longlong, [C.c_int32, C.c_int32, C.c_int32]),
    "sp_reduce_publish": (
        C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int64, C.c_void_p]
    ),
    "sp_reduce_combine": (
        C.c_int,
        [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p,
         C.c_void_p],
    ),
    "sp_mailbox_create": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_void_p)]),
    "sp_mailbox_destroy": (C.c_int, [C.c_void_p]),
    "sp_ipc_get_handle": (C.c_int, [C.c_void_p, C.c_void_p]),
    "sp_ipc_open_handle": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "sp_ipc_close_handle": (C.c_int, [C.c_void_p]),
    "sp_op_attention": (
        C.c_int,
        [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
         C.c_int32, C.c_void_p],
    ),
}

_lock = threading.Lock()
_lib: C.CDLL | None = None


def library_path() -> Path:
    return LIB_PATH


def load() -> C.CDLL:
    """Load (once) the engine library; raises RuntimeError if it is absent or incompatible."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"CUDA engine library {LIB_PATH} is missing: run `python -m paper_2408_12526_b200.build` "
                "(there is no CPU fallback)"
            )
        lib = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.sp_abi_version() != ABI_VERSION:
            raise RuntimeError(f"engine ABI {lib.sp_abi_version()} != expected {ABI_VERSION}")
        _lib = lib
        return lib


def check(rc: int) -> None:
    """Map an sp_status to the exception the reference would raise."""
    if rc == SP_OK:
        return
    msg = (load().sp_last_error() or b"").decode(errors="replace")
    if rc == SP_EINVAL:
        raise ValueError(msg)
    if rc == SP_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(f"CUDA engine failure: {msg}")

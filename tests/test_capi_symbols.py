"""The C-ABI library loads on CPU and exports every symbol include/studentpar_b200.h declares
(no compute calls: there is no GPU here)."""
import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "studentpar_b200.h"


def declared_symbols():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(sp_[a-z_0-9]+)\s*\(", text)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for must in ["sp_group_create", "sp_group_destroy", "sp_group_forward", "sp_group_forward_dense",
                 "sp_group_forward_host", "sp_last_error", "sp_abi_version"]:
        assert must in syms


def test_library_exports_every_declared_symbol():
    from paper_2408_12526_b200 import _lib
    from paper_2408_12526_b200.build import LIB_PATH, build

    if not LIB_PATH.exists():
        build()
    lib = ctypes.CDLL(str(LIB_PATH))
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, f"symbols declared but not exported: {missing}"
    # the Python binding covers exactly the declared surface
    assert sorted(_lib.SIGNATURES) == declared_symbols()


def test_abi_version_and_error_path_without_gpu():
    from paper_2408_12526_b200 import _lib

    lib = _lib.load()
    assert lib.sp_abi_version() == _lib.ABI_VERSION
    # argument validation happens before any CUDA call: a NULL config is a ValueError
    handle = ctypes.c_void_p()
    rc = lib.sp_group_create(None, None, 0, ctypes.byref(handle))
    assert rc == _lib.SP_EINVAL
    with pytest.raises(ValueError):
        _lib.check(rc)
    assert b"null" in lib.sp_last_error()


def test_engine_refuses_cpu_fallback():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2408_12526_b200 import StudentGroup, random_dense_group

    with pytest.raises(RuntimeError, match="no CPU fallback"):
        StudentGroup(random_dense_group(8, 16, 2, 2))


def test_torch_extension_registers_the_ops():
    """The thin PyTorch C++ extension (csrc/sp_torch.cpp) loads without a GPU and registers
    torch.ops.studentpar.{group_forward, group_forward_graph, group_forward_host}; a null handle is
    rejected before any CUDA call."""
    import torch

    from paper_2408_12526_b200.build import TORCH_LIB_PATH, build
    from paper_2408_12526_b200.group import torch_ops

    if not TORCH_LIB_PATH.exists():
        build()
    ops = torch_ops()
    assert ops is not None
    for name in ("group_forward", "group_forward_graph", "group_forward_host"):
        assert hasattr(ops, name)
    with pytest.raises(RuntimeError, match="null group handle"):
        ops.group_forward_host(0, torch.zeros(1, dtype=torch.int32), torch.tensor([0, 1], dtype=torch.int32), 1,
                               torch.zeros(1, 2), True, 0)

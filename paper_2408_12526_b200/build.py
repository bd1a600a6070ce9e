"""Build the sm_100a C-ABI library in-tree (nvcc; no torch headers, no JIT cache).

    python -m paper_2408_12526_b200.build          # incremental
    python -m paper_2408_12526_b200.build --force  # full rebuild

Output: paper_2408_12526_b200/_lib/libstudentpar_b200.so (git-ignored, travels with gpurun).
"""
from __future__ import annotations

import argparse
import os
import shutil
import subprocess
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
INCLUDE = PKG.parent / "include"
OUT_DIR = PKG / "_lib"
OBJ_DIR = OUT_DIR / "obj"
LIB_NAME = "libstudentpar_b200.so"
LIB_PATH = OUT_DIR / LIB_NAME
TORCH_LIB_PATH = OUT_DIR / "libstudentpar_torch.so"  # torch.ops.studentpar (sp_torch.cpp)

ARCH_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "--expt-relaxed-constexpr"]


def _nvcc() -> str:
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(cand):
        raise RuntimeError("nvcc not found; the CUDA extension cannot be built")
    return cand


def _sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu"))


def _headers() -> list[Path]:
    return sorted(CSRC.glob("*.cuh")) + sorted(INCLUDE.glob("*.h"))


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def _torch_flags() -> tuple[list[str], list[str]]:
    import torch
    from torch.utils import cpp_extension as ce

    abi = int(torch._C._GLIBCXX_USE_CXX11_ABI)
    cuda_inc = str(Path(_nvcc()).resolve().parent.parent / "include")
    cflags = [f"-D_GLIBCXX_USE_CXX11_ABI={abi}", "-I", cuda_inc] + [f for p in ce.include_paths() for f in ("-I", p)]
    libdir = ce.library_paths()[0]
    ldflags = ["-L", libdir, "-Wl,-rpath," + libdir, "-lc10", "-lc10_cuda", "-ltorch_cpu", "-ltorch_cuda",
               "-L", str(OUT_DIR), "-Wl,-rpath,$ORIGIN", "-lstudentpar_b200"]
    return cflags, ldflags


def build_torch_ops(force: bool = False) -> Path:
    """The thin PyTorch C++ extension (csrc/sp_torch.cpp) over the C ABI -> _lib/libstudentpar_torch.so."""
    src = CSRC / "sp_torch.cpp"
    if not force and not _stale(TORCH_LIB_PATH, [src, LIB_PATH] + sorted(INCLUDE.glob("*.h"))):
        return TORCH_LIB_PATH
    cflags, ldflags = _torch_flags()
    tmp = TORCH_LIB_PATH.with_suffix(".so.tmp")
    cmd = [shutil.which("g++") or "g++", "-O2", "-std=c++17", "-shared", "-fPIC", *cflags, str(src), "-o", str(tmp),
           *ldflags]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"g++ failed:\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, TORCH_LIB_PATH)
    return TORCH_LIB_PATH


def build(force: bool = False, verbose: bool = False) -> Path:
    OBJ_DIR.mkdir(parents=True, exist_ok=True)
    nvcc = _nvcc()
    headers = _headers()
    jobs = []
    objs = []
    for src in _sources():
        obj = OBJ_DIR / (src.stem + ".o")
        objs.append(obj)
        if force or _stale(obj, [src] + headers):
            cmd = [nvcc, *ARCH_FLAGS, *NVCC_FLAGS, "-I", str(INCLUDE), "-c", str(src), "-o", str(obj)]
            if verbose:
                cmd.insert(1, "-Xptxas=-v")
            jobs.append(cmd)

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed:\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        if verbose and (r.stdout or r.stderr):
            print(r.stdout + r.stderr)

    with ThreadPoolExecutor(max_workers=min(8, max(1, len(jobs)))) as ex:
        list(ex.map(run, jobs))
    if force or jobs or _stale(LIB_PATH, objs):
        tmp = LIB_PATH.with_suffix(".so.tmp")
        cmd = [nvcc, *ARCH_FLAGS, "-shared", "-o", str(tmp), *map(str, objs)]
        run(cmd)
        os.replace(tmp, LIB_PATH)
    build_torch_ops(force)
    return LIB_PATH


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", "--verbose", action="store_true")
    args = ap.parse_args()
    print(build(force=args.force, verbose=args.verbose))


if __name__ == "__main__":
    main()

"""Build libtacsl_b200.so in-tree with nvcc for sm_100a (B200).

    python -m paper_2408_06506_b200.build [--verbose]

The library is a plain C-ABI shared object (include/tacsl_b200.h): it links
the CUDA runtime statically and has no torch dependency, so the ctypes layer
(paper_2408_06506_b200/_lib.py) and any other FFI can load it.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
INCLUDE = ROOT / "include"
LIB_NAME = "libtacsl_b200.so"
LIB_PATH = PKG / LIB_NAME

ARCH_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [
    "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
    "-DTACSL_BUILD",
]


def nvcc_path() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; the tacsl_b200 kernels need CUDA 12.9+ nvcc for sm_100a")


def sources():
    return sorted(CSRC.glob("*.cu"))


def needs_rebuild() -> bool:
    if not LIB_PATH.exists():
        return True
    mtime = LIB_PATH.stat().st_mtime
    deps = list(sources()) + list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + list(INCLUDE.glob("*.h"))
    return any(p.stat().st_mtime > mtime for p in deps)


def build(verbose: bool = False, force: bool = False) -> Path:
    """Compile every csrc/*.cu to an object in parallel (one nvcc per file),
    then link the shared library; the .so is replaced atomically."""
    if not force and not needs_rebuild():
        return LIB_PATH
    from concurrent.futures import ThreadPoolExecutor

    nvcc = nvcc_path()
    objdir = PKG / "build_obj"
    objdir.mkdir(exist_ok=True)
    flags = [*ARCH_FLAGS, *NVCC_FLAGS, f"-I{INCLUDE}", f"-I{CSRC}"]
    if verbose:
        flags.insert(0, "-Xptxas=-v")

    def compile_one(src: Path):
        obj = objdir / (src.stem + ".o")
        cmd = [nvcc, *flags, "-c", str(src), "-o", str(obj)]
        if verbose:
            print(" ".join(cmd), flush=True)
        return obj, subprocess.run(cmd, capture_output=True, text=True)

    srcs = list(sources())
    with ThreadPoolExecutor(max_workers=min(len(srcs), os.cpu_count() or 1)) as ex:
        results = list(ex.map(compile_one, srcs))
    failed = False
    for obj, res in results:
        if verbose or res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
        failed |= res.returncode != 0
    if failed:
        raise RuntimeError(f"nvcc failed building {LIB_NAME}")
    tmp = LIB_PATH.with_suffix(".so.tmp")
    cmd = [nvcc, *ARCH_FLAGS, "-shared", "-o", str(tmp), *(str(o) for o, _ in results)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if verbose or res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed ({res.returncode}) linking {LIB_NAME}")
    os.replace(tmp, LIB_PATH)
    shutil.rmtree(objdir, ignore_errors=True)
    return LIB_PATH


if __name__ == "__main__":
    p = build(verbose="--verbose" in sys.argv, force="--force" in sys.argv)
    print(p)

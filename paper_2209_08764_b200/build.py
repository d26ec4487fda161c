"""Build libs3bfs.so in-tree with nvcc for sm_100a (no JIT cache, no pip install)."""
from __future__ import annotations

import os
import shutil
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libs3bfs.so")
LIB_CHECK = os.path.join(HERE, "libs3bfs_check.so")  # S3BFS_CHECK=1: bounds-checked build
SOURCES = [os.path.join(CSRC, "s3bfs.cu")]
DEPS = SOURCES + [os.path.join(CSRC, "s3bfs_kernels.cuh"), os.path.join(ROOT, "include", "s3bfs.h")]

NVCC_FLAGS = [
    "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
    "-Xcompiler", "-fPIC", "-shared",
]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: the CUDA path cannot be built")


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in DEPS)


def build(force: bool = False, verbose: bool = False, defines=(), out: str = LIB) -> str:
    """Compile libs3bfs.so (or a design variant with -D defines, for experiments only)."""
    if out == LIB and not defines and not force and not stale():
        return LIB
    tmp = out + f".tmp{os.getpid()}"
    cmd = [nvcc(), *NVCC_FLAGS, *(["-Xptxas", "-v"] if verbose else []),
           *[f"-D{d}" for d in defines], "-o", tmp, *SOURCES]
    subprocess.check_call(cmd, cwd=HERE)
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    print(build(force=True, verbose=True))

"""Build kx_micro variant libraries into variants/ (experiment harness)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
V = {
    "base": [], "norank": ["S3BFS_KX_RANK=0"],
    "novec": ["S3BFS_KX_VEC=0"], "vec16": ["S3BFS_KX_GROUPS=16"],
    "nofast": ["S3BFS_KX_FAST=0"], "bmca": ["S3BFS_BM_NC=0"],
    "g4": ["S3BFS_KX_GROUPS=4"],
    "g16": ["S3BFS_KX_GROUPS=16"], "t1024": ["S3BFS_KD_THREADS=1024"],
    "g8m3": ["S3BFS_KD_MINB=3"], "g4m3": ["S3BFS_KX_GROUPS=4", "S3BFS_KD_MINB=3"],
    "g4m4": ["S3BFS_KX_GROUPS=4", "S3BFS_KD_MINB=4"], "g2m4": ["S3BFS_KX_GROUPS=2", "S3BFS_KD_MINB=4"],
    "g6m3": ["S3BFS_KX_GROUPS=6", "S3BFS_KD_MINB=3"],
}
sel = sys.argv[1:] or list(V)
os.makedirs(os.path.join(ROOT, "variants"), exist_ok=True)
for k in sel:
    out = os.path.join(ROOT, "variants", f"libkx_{k}.so")
    cmd = ["nvcc", "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
           "-Xcompiler", "-fPIC", "-shared", *[f"-D{d}" for d in V[k]], "-o", out,
           os.path.join(ROOT, "scripts", "kx_micro.cu")]
    subprocess.check_call(cmd)
    print(k, out)

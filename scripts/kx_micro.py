"""Experiment driver (not a benchmark line): time k_explore variants on captured levels.
usage: python scripts/kx_micro.py CONFIG SRC_INDEX tag=lib.so ...  (libs from build_micro)"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import graphgen  # noqa: E402
import paper_2209_08764_b200 as pkg  # noqa: E402

cfg, si = sys.argv[1], int(sys.argv[2])
relabel = os.environ.get("RELABEL", "0") == "1"
g = graphgen.make_config(cfg)
dev = torch.device("cuda")
ro = torch.from_numpy(g.row_offsets).to(dev)
col = torch.from_numpy(g.col_indices).to(dev)
n = g.n
bfs = pkg.S3BFS(ro, col)
s = g.sources[si]
lvl, par = bfs.run(s)
torch.cuda.synchronize()
deg = (ro[1:] - ro[:-1])
if relabel:  # degree-descending internal ids (experiment: hot vertices get the lowest ids)
    n2o = torch.sort(deg, descending=True, stable=True).indices
    o2n = torch.empty_like(n2o)
    o2n[n2o] = torch.arange(n, device=dev)
    deg2 = deg[n2o]
    ro2 = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    ro2[1:] = torch.cumsum(deg2.long(), 0)
    idx = torch.repeat_interleave(ro[:-1][n2o].long() - ro2[:-1], deg2.long()) + \
        torch.arange(g.nnz, device=dev)
    col = o2n[col[idx].long()].to(torch.int32).contiguous()
    del idx
    ro = ro2.to(torch.int32)
    lvl = lvl[n2o]
    deg = deg2
    torch.cuda.synchronize()
col = torch.cat([col, torch.zeros(1024, dtype=torch.int32, device=dev)])  # vector over-read pad
L = int(lvl.max().item())
lpbuf = torch.zeros((n, 2), dtype=torch.int32, device=dev)
vinfo = torch.zeros((n, 4), dtype=torch.int32, device=dev)
vinfo[:, 0] = ro[:-1]
vinfo[:, 1] = deg
cand = torch.empty(g.nnz + 1_000_000, dtype=torch.int32, device=dev)
wcnt = torch.zeros(4096 * 64, dtype=torch.int32, device=dev)
status = torch.zeros(4096, dtype=torch.int64, device=dev)
claim = torch.zeros(max(16, 1 << (n - 1).bit_length()), dtype=torch.uint8, device=dev)  # pow2 slots
out_l = torch.empty(n, dtype=torch.int32, device=dev)
out_p = torch.empty(n, dtype=torch.int32, device=dev)
levels = []
for l in range(L + 1):
    fr = torch.nonzero(lvl == l).flatten().to(torch.int32)
    e_l = int(deg[fr.long()].sum().item())
    if e_l > 5_000_000:
        levels.append((l, fr, e_l))
libs = [a.split("=", 1) for a in sys.argv[3:]]
for l, fr, e_l in levels:
    visited = (lvl >= 0) & (lvl <= l)
    bits = torch.zeros((n + 127) // 128 * 128, dtype=torch.int64, device=dev)
    bits[:n] = visited.to(torch.int64)
    w = (bits.view(-1, 32) << torch.arange(32, device=dev, dtype=torch.int64)).sum(1)
    bm = w.to(torch.int64).to(torch.int32)  # two's complement view of the u32 words
    bm = torch.cat([bm, torch.full((4,), -1, dtype=torch.int32, device=dev)])  # sentinel block
    for order in ("discovery", "sorted"):
        f = fr if order == "sorted" else fr[torch.randperm(fr.numel(), device=dev)]
        f = f.contiguous()
        d = deg[f.long()]
        fex = torch.zeros(f.numel() + 1, dtype=torch.int32, device=dev)
        fex[1:] = torch.cumsum(d, 0).to(torch.int32)
        frs = ro[f.long()].contiguous()
        raw = ctypes.CDLL(os.path.abspath(libs[0][1]))
        raw.kx_raw.argtypes = [ctypes.c_void_p, ctypes.c_longlong, ctypes.c_void_p, ctypes.c_void_p,
                               ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                               ctypes.POINTER(ctypes.c_float)]
        for which, name in ((0, "stream-all-col"), (1, "rows-warp"), (2, "rows-warp+bm"),
                            (3, "rows-chunked"), (4, "rows-chunked+bm")):
            if which == 0 and order == "sorted":
                continue
            ms = ctypes.c_float()
            raw.kx_raw(col.data_ptr(), g.nnz, frs.data_ptr(), fex.data_ptr(), f.numel(),
                       bm.data_ptr(), which, 5, ctypes.byref(ms))
            arcs = g.nnz if which == 0 else e_l
            print(f"L{l} {order:9s} raw {name:16s} {ms.value*1e3:8.1f} us  "
                  f"{arcs*4/ms.value/1e6:7.1f} GB/s of col  {arcs/ms.value/1e6:7.1f} Garcs/s", flush=True)
        for tag, path in libs:
            lib = ctypes.CDLL(os.path.abspath(path))
            ms = ctypes.c_float()
            cands = ctypes.c_int()
            vp = ctypes.c_void_p
            lib.kx_micro.argtypes = [vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, vp, vp, vp, vp,
                                     vp, vp, vp, vp, vp, vp, vp, vp, ctypes.c_int, ctypes.c_int,
                                     ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_float),
                                     ctypes.POINTER(ctypes.c_int)]
            rc = lib.kx_micro(col.data_ptr(), n, f.numel(), e_l, f.data_ptr(), frs.data_ptr(),
                              fex.data_ptr(), bm.data_ptr(), claim.data_ptr(), vinfo.data_ptr(),
                              lpbuf.data_ptr(),
                              out_l.data_ptr(), out_p.data_ptr(), cand.data_ptr(),
                              wcnt.data_ptr(), status.data_ptr(), 296, 16384, l, 5,
                              ctypes.byref(ms), ctypes.byref(cands))
            print(f"L{l} e_l={e_l/1e6:7.1f}M n_l={f.numel()/1e6:5.2f}M {order:9s} {tag:14s} "
                  f"{ms.value*1e3:8.1f} us  {e_l/ms.value/1e6:7.1f} Garcs/s  cand={cands.value} rc={rc}",
                  flush=True)

"""Test-only numpy stand-in for one NEXT-4 rank (paper_2209_08764_b200.dist.DistRank).

It has the library's per-level semantics (include/s3bfs.h, NEXT-4): rank r of G explores the
global edges [r*e_l/G, (r+1)*e_l/G) of the level (frontier order, row order), keeps the first
discovery of each unvisited vertex (its own dedup), and hands out records {v, parent, row
start, degree}; merge keeps each vertex from the lowest rank, in rank-major record order.
It lets the CPU tests run the real driver (dist.traverse) and the real collectives (gloo)
without a GPU.  Not product code; shares nothing with oracle/.
"""
import numpy as np
import torch


class NumpyRank:
    def __init__(self, row_offsets, col_indices, rank, size):
        self.ro = np.asarray(row_offsets, dtype=np.int64)
        self.col = np.asarray(col_indices, dtype=np.int64)
        self.n = len(self.ro) - 1
        self.rank, self.size = rank, size
        self.device = torch.device("cpu")

    def begin(self, source):
        self.level = np.full(self.n, -1, dtype=np.int32)
        self.parent = np.full(self.n, -1, dtype=np.int32)
        self.level[source], self.parent[source] = 0, source
        self.frontier = [source]
        self.l = 0
        self.rec = []

    def expand(self):
        deg = [int(self.ro[x + 1] - self.ro[x]) for x in self.frontier]
        e_l = sum(deg)
        if not self.frontier or e_l == 0:
            return 0, True
        lo = e_l * self.rank // self.size
        hi = e_l * (self.rank + 1) // self.size
        seen, self.rec, e = set(), [], 0
        for x, d in zip(self.frontier, deg):
            for k in range(d):
                if lo <= e < hi:
                    v = int(self.col[self.ro[x] + k])
                    if self.level[v] < 0 and v not in seen:
                        seen.add(v)
                        self.rec.append((v, x, int(self.ro[v]), int(self.ro[v + 1] - self.ro[v])))
                e += 1
        return len(self.rec), False

    def records(self, n_local, stride):
        buf = torch.zeros((stride, 4), dtype=torch.int32)
        if n_local:
            buf[:n_local] = torch.tensor(self.rec[:n_local], dtype=torch.int32)
        return buf

    def merge(self, all_records, counts, stride):
        a = all_records.numpy()
        nxt = []
        for r, c in enumerate(counts):
            for i in range(c):
                v, p = int(a[r * stride + i, 0]), int(a[r * stride + i, 1])
                if self.level[v] < 0:
                    self.level[v], self.parent[v] = self.l + 1, p
                    nxt.append(v)
        self.frontier = nxt
        self.l += 1

    def end(self):
        return self.level, self.parent

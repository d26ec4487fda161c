"""Test-only numpy stand-in for one NEXT-4 rank (paper_2209_08764_b200.dist.DistRank).

It has the library's per-level semantics (include/s3bfs.h, NEXT-4, 1-D vertex partition):
rank r of G owns the vertices v with (v // 32) % G == r; it explores the rows of its own
frontier vertices, sends every target whose (replicated) visited flag is clear -- once per
level -- to the target's owner, keeps one received copy of each of its own unvisited vertices
(the Owner check), and publishes its new vertices' visited flags to every rank.  Where the
library moves data by peer stores, the stand-in uses the group's collectives (gloo) or, in
one process, the peer objects directly.  It lets the CPU tests run the real driver
(dist.traverse) and real collectives without a GPU.  Not product code; shares nothing with
oracle/.
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
        self.peers = None

    def owner(self, v):
        return (v // 32) % self.size

    def export(self):
        return self.rank  # in a process group the stand-in talks through the collectives

    def connect(self, peers, use_ipc):  # noqa: D401
        self.peers = peers  # loopback: the peer objects themselves

    def begin(self, source):
        self.visited = np.zeros(self.n, dtype=bool)
        self.visited[source] = True
        self.level = np.full(self.n, -1, dtype=np.int32)
        self.parent = np.full(self.n, -1, dtype=np.int32)
        self.frontier = []
        if self.owner(source) == self.rank:
            self.level[source], self.parent[source] = 0, source
            self.frontier = [source]
        self.l = 0

    def explore(self):
        self.out = [[] for _ in range(self.size)]
        sent = set()
        for x in self.frontier:
            for k in range(self.ro[x], self.ro[x + 1]):
                v = int(self.col[k])
                if not self.visited[v] and v not in sent:
                    sent.add(v)
                    self.out[self.owner(v)].append((v, x))
        self.inbox = []

    def exchange(self, group):
        if group is None:
            for d, lst in enumerate(self.out):
                self.peers[d].inbox.extend(lst)
            return
        import torch.distributed as dist
        allout = [None] * self.size
        dist.all_gather_object(allout, self.out, group=group)
        self.inbox = [it for src in range(self.size) for it in allout[src][self.rank]]

    def dedup(self):
        self.next = []
        for v, p in self.inbox:
            if self.level[v] < 0:
                self.level[v], self.parent[v] = self.l + 1, p
                self.next.append(v)

    def publish(self, group):
        if group is None:
            for q in self.peers:
                q.visited[self.next] = True
            return
        import torch.distributed as dist
        allnew = [None] * self.size
        dist.all_gather_object(allnew, self.next, group=group)
        for lst in allnew:
            self.visited[lst] = True

    def advance(self, group):
        if group is None:
            total = sum(len(q.next) for q in self.peers)
        else:
            import torch.distributed as dist
            t = torch.tensor([len(self.next)], dtype=torch.int64)
            dist.all_reduce(t, group=group)
            total = int(t.item())
        self.frontier = self.next
        self.l += 1
        return total == 0, total

    def end(self):
        return torch.from_numpy(self.level.copy()), torch.from_numpy(self.parent.copy())

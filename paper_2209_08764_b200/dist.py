"""NEXT-4 ("distributed settings"): one traversal over G ranks.

Replicated-graph split: every rank holds the whole graph and the same frontier, explores
1/G of each level's edges with the single-GPU kernels, and deduplicates its own discoveries
(Owner check).  The exchange step of a level is an all-gather of every rank's kept vertices
(records {internal id, parent, row start, degree}); ``s3bfs_dist_merge`` then keeps each
vertex once (lowest rank) and builds the identical next frontier on every rank.  All of the
path's arithmetic runs in the library's kernels; this module is plumbing: the level loop and
the collectives (``torch.distributed`` all-gathers -- NCCL over NVLink on a multi-GPU node).

``traverse(ranks, source, group)`` drives the protocol for the ranks held by this process:
one ``DistRank`` per process in a process group, or several ``DistRank`` objects in one
process with ``group=None`` (loopback: the "all-gather" is a concatenation).  Any object with
the ``DistRank`` methods can stand in for a rank (the CPU tests use a numpy stand-in to
check the protocol on a gloo group).
"""
from __future__ import annotations

from . import s3bfs as _s


class DistRank:
    """Rank ``rank`` of ``size``: a dist handle over device CSR tensors (kept alive here)."""

    def __init__(self, row_offsets, col_indices, rank: int, size: int,
                 options: _s.Options | None = None, stream=None):
        import torch
        # a copy: the caller's options object is never turned into a dist configuration
        o = _s.Options() if options is None else _s.Options.from_buffer_copy(options)
        o.dist_size, o.dist_rank = int(size), int(rank)
        self.rank, self.size = int(rank), int(size)
        self.row_offsets, self.col_indices = row_offsets, col_indices
        self.n = row_offsets.numel() - 1
        self.device = row_offsets.device
        self.stream = stream
        self.handle = _s.s3bfs_create(row_offsets, col_indices, o, stream)
        self.level = torch.empty(self.n, dtype=torch.int32, device=self.device)
        self.parent = torch.empty(self.n, dtype=torch.int32, device=self.device)

    # -- the five protocol steps (include/s3bfs.h, NEXT-4) --
    def begin(self, source: int) -> None:
        _s.s3bfs_dist_begin(self.handle, source, self.level, self.parent, self.stream)

    def expand(self) -> tuple[int, bool]:
        return _s.s3bfs_dist_expand(self.handle, self.stream)

    def records(self, n_local: int, stride: int):
        import torch
        buf = torch.zeros((max(stride, 1), 4), dtype=torch.int32, device=self.device)
        _s.s3bfs_dist_records(self.handle, buf, n_local, self.stream)
        return buf[:stride]

    def merge(self, all_records, counts, stride: int) -> None:
        _s.s3bfs_dist_merge(self.handle, all_records.contiguous(), counts, stride, self.stream)

    def end(self):
        _s.s3bfs_dist_end(self.handle, self.stream)
        return self.level, self.parent

    def close(self) -> None:
        if self.handle:
            _s.s3bfs_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


def _gather_counts(local: list[int], group, device) -> list[int]:
    if group is None:
        return list(local)
    import torch
    import torch.distributed as dist
    assert len(local) == 1, "one rank per process in a process group"
    t = torch.tensor(local, dtype=torch.int64, device=device)
    out = [torch.zeros_like(t) for _ in range(dist.get_world_size(group))]
    dist.all_gather(out, t, group=group)
    return [int(x.item()) for x in out]


def _gather_records(send: list, group):
    import torch
    if group is None:
        return torch.cat(send, 0)
    import torch.distributed as dist
    out = [torch.empty_like(send[0]) for _ in range(dist.get_world_size(group))]
    dist.all_gather(out, send[0].contiguous(), group=group)
    return torch.cat(out, 0)


def traverse(ranks: list, source: int, group=None) -> list:
    """Run one traversal from `source`; returns [(level, parent)] of the local ranks.

    Every rank of the job must call this with the same source.  The loop ends on every rank
    at the same level: the merged frontier, hence the done flag, is identical everywhere."""
    for r in ranks:
        r.begin(source)
    levels = 0
    while True:
        st = [r.expand() for r in ranks]
        done = {d for _, d in st}
        if len(done) != 1:
            raise RuntimeError("ranks disagree on termination (frontiers diverged)")
        if done.pop():
            break
        local = [nl for nl, _ in st]
        counts = _gather_counts(local, group, ranks[0].device)
        stride = max(counts)
        send = [r.records(nl, stride) for r, nl in zip(ranks, local)]
        allrec = _gather_records(send, group)
        for r in ranks:
            r.merge(allrec, counts, stride)
        levels += 1
    return [r.end() for r in ranks]

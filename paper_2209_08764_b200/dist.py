"""NEXT-4 ("distributed settings"): one traversal over G ranks.

1-D vertex partition: rank r owns the internal ids v with (v / 32) mod G == r, their CSR rows
and their state (include/s3bfs.h, NEXT-4).  Per level every rank explores its own frontier;
a target whose visited bit (replicated bitmap) is clear is stored as {v, parent} straight into
v's owner's receive segment -- peer memory over NVLink, written by the exploration kernel
itself; the owner deduplicates (Owner check on its own GPU), publishes its new visited words
and its totals into every peer, and the totals over all ranks end the loop.  All of the path's
arithmetic and all data movement run in the library's kernels; this module is plumbing: the
connection (exchange records, CUDA IPC between processes), the phase order and the final
combination of the ranks' answers.

``traverse(ranks, source, group)`` drives the protocol for the ranks held by this process:
one ``DistRank`` per process of a process group (``connect(ranks, group)`` first), or several
``DistRank`` objects in one process with ``group=None`` (a loopback on one GPU: the ranks run
their phases in turn, so no kernel ever waits for another rank's kernel).  Between the phases
a process group runs a one-element all-reduce on the current stream: a stream-ordered barrier
(NCCL on GPUs), no host round trip.  Any object with the ``DistRank`` methods can stand in
for a rank (the CPU tests use a numpy stand-in on a gloo group).
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

    # -- connection --
    def export(self):
        return _s.s3bfs_dist_export(self.handle)

    def connect(self, peers, use_ipc: bool) -> None:
        _s.s3bfs_dist_connect(self.handle, peers, use_ipc)

    # -- the per-level protocol (include/s3bfs.h, NEXT-4) --
    def begin(self, source: int) -> None:
        _s.s3bfs_dist_begin(self.handle, source, self.level, self.parent, self.stream)

    def explore(self) -> None:
        _s.s3bfs_dist_explore(self.handle, self.stream)

    def exchange(self, group) -> None:
        """Nothing to move: the explore kernel stored the candidates in the owners' memory."""

    def dedup(self) -> None:
        _s.s3bfs_dist_dedup(self.handle, self.stream)

    def publish(self, group) -> None:
        """Nothing to move: the dedup kernels stored the bitmap words and totals in the peers."""

    def advance(self, group, wait: bool = True):
        """Advance the level; with wait: (done, next frontier size over all ranks)."""
        return _s.s3bfs_dist_advance(self.handle, self.stream, wait=wait)

    def advance_flag(self, flag_ptr: int) -> None:
        """Advance without a host round trip; the device writes -1 (done) or the next frontier
        size over all ranks into the int64 at flag_ptr (pinned host memory)."""
        _s.s3bfs_dist_advance_flag(self.handle, flag_ptr, self.stream)

    def status(self) -> tuple[bool, int]:
        return _s.s3bfs_dist_status(self.handle, self.stream)

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


def connect(ranks: list, group=None) -> None:
    """Give every rank the exchange records of all ranks (rank order).  group=None: the ranks
    are all in this process (addresses used as they are); otherwise one rank per process, the
    records travel through the group and peers' allocations are opened by CUDA IPC."""
    if group is None:
        peers = [r.export() for r in ranks]
        if not all(isinstance(p, _s.DistPeer) for p in peers):
            peers = list(ranks)  # stand-ins (tests) exchange through each other directly
        for r in ranks:
            r.connect(peers, use_ipc=False)
        return
    import ctypes

    import torch.distributed as dist
    assert len(ranks) == 1, "one rank per process in a process group"
    mine = ranks[0].export()
    if isinstance(mine, ctypes.Structure):  # a library record travels as its bytes
        mine = bytes(mine)
    allrec = [None] * dist.get_world_size(group)
    dist.all_gather_object(allrec, mine, group=group)
    peers = [_s.DistPeer.from_buffer_copy(b) if isinstance(b, (bytes, bytearray)) else b
             for b in allrec]
    ranks[0].connect(peers, use_ipc=True)


def _barrier(ranks, group) -> None:
    """Order the phases across ranks.  One process: the ranks' work was enqueued in phase order
    (same stream), nothing to do.  A group: a one-element all-reduce on the current stream."""
    if group is None:
        return
    import torch
    import torch.distributed as dist
    t = torch.zeros(1, dtype=torch.int32, device=ranks[0].device)
    dist.all_reduce(t, group=group)


def _combine(outs, group):
    """Every rank wrote its own vertices and -1 elsewhere: the element-wise max is the answer."""
    if group is None:
        import numpy as np
        lv, pa = outs[0]
        for a, b in outs[1:]:
            if isinstance(lv, np.ndarray):
                lv, pa = np.maximum(lv, a), np.maximum(pa, b)
            else:
                import torch
                lv, pa = torch.maximum(lv, a), torch.maximum(pa, b)
        return [(lv, pa) for _ in outs]
    import torch
    import torch.distributed as dist
    (lv, pa), = outs
    lv_t = lv if isinstance(lv, torch.Tensor) else torch.from_numpy(lv)
    pa_t = pa if isinstance(pa, torch.Tensor) else torch.from_numpy(pa)
    dist.all_reduce(lv_t, op=dist.ReduceOp.MAX, group=group)
    dist.all_reduce(pa_t, op=dist.ReduceOp.MAX, group=group)
    return [(lv_t, pa_t)]


def traverse(ranks: list, source: int, group=None, lag: int = 2) -> list:
    """Run one traversal from `source`; returns [(level, parent)] (the full answer) for the
    local ranks.  Every rank of the job must call this with the same source; the loop ends on
    every rank at the same level (the totals over all ranks decide).

    Library ranks: the levels are enqueued without a host round trip -- each level's advance
    writes its termination flag into pinned host memory and the host reads the flag of the
    level `lag` levels back (behind a CUDA event), so up to `lag` levels past the end are
    enqueued; they are no-ops on the device.  Stand-ins without advance_flag advance with
    a host read per level."""
    for r in ranks:
        r.begin(source)
    if all(hasattr(r, "advance_flag") for r in ranks):
        _levels_flagged(ranks, group, max(lag, 0))
        return _combine([r.end() for r in ranks], group)
    levels = 0
    while True:
        for r in ranks:
            r.explore()
        for r in ranks:
            r.exchange(group)
        _barrier(ranks, group)
        for r in ranks:
            r.dedup()
        for r in ranks:
            r.publish(group)
        _barrier(ranks, group)
        st = [r.advance(group) for r in ranks]
        done = {d for d, _ in st}
        if len(done) != 1:
            raise RuntimeError("ranks disagree on termination")
        levels += 1
        if done.pop():
            break
    return _combine([r.end() for r in ranks], group)


def _levels_flagged(ranks: list, group, lag: int) -> None:
    import torch
    slots = torch.zeros((lag + 1, len(ranks)), dtype=torch.int64).pin_memory()
    pending = []  # (level, event) whose flags are not read yet
    lv = 0
    while True:
        for r in ranks:
            r.explore()
        for r in ranks:
            r.exchange(group)
        _barrier(ranks, group)
        for r in ranks:
            r.dedup()
        for r in ranks:
            r.publish(group)
        _barrier(ranks, group)
        k = lv % (lag + 1)
        for i, r in enumerate(ranks):
            r.advance_flag(slots[k, i].data_ptr())
        ev = torch.cuda.Event()
        ev.record()
        pending.append((lv, ev))
        lv += 1
        if len(pending) > lag:
            old, e = pending.pop(0)
            e.synchronize()
            flags = slots[old % (lag + 1)].tolist()
            done = {f == -1 for f in flags}
            if len(done) != 1:
                raise RuntimeError("ranks disagree on termination")
            if done.pop():
                return

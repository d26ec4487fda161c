"""The N>1 bench path on CPU: world-size-2 gloo processes run the same sharding and
max-over-ranks / sum-over-ranks reductions bench.py uses under torchrun (replicas only:
independent sources, no data-path collective -- DESIGN.md s.9)."""
import os
import socket
import sys

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    sys.path.insert(0, ROOT)
    import bench
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    srcs = list(range(100, 116))
    mine = bench.shard_sources(srcs, rank, world)
    # per-rank device time and edges (rank-dependent so the reductions are checked)
    gteps, max_ms, tot = bench.job_throughput(10.0 + rank, 1e9 * (rank + 1), "cpu", world)
    out[rank] = (mine, gteps, max_ms, tot)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_sharding_and_reductions():
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
        res = dict(out)
    m0, m1 = res[0][0], res[1][0]
    assert sorted(m0) == sorted(m1) == list(range(100, 116))   # each rank: every source once
    assert m0[0] != m1[0]                                       # different traversal order
    for r in (0, 1):
        _, gteps, max_ms, tot = res[r]
        assert max_ms == 11.0                                   # max over ranks
        assert tot == 3e9                                       # sum over ranks
        assert abs(gteps - 3e9 / 0.011 / 1e9) < 1e-9


def test_single_rank_is_plain():
    sys.path.insert(0, ROOT)
    import bench
    g, ms, tot = bench.job_throughput(2.0, 4e9, "cpu", 1)
    assert ms == 2.0 and tot == 4e9 and abs(g - 2000.0) < 1e-9
    assert bench.shard_sources([1, 2, 3], 0, 1) == [1, 2, 3]


def test_launch_count_from_tier_sequence():
    """bench.py's gpu_launches: k_init + one k_small per tier-0 run + one k_cluster per
    cluster run + 2 per top-down level + 3 per bottom-up level + k_finalize (tier 2 = a last
    level with nothing to explore launches nothing)."""
    sys.path.insert(0, ROOT)
    import numpy as np
    import bench
    st = {"tier": np.array([0, 0, 4, 4, 1, 1, 3, 1, 4, 0, 0, 2])}
    assert bench.launches_from_stats(st) == 1 + 2 + 2 + 2 * 3 + 3 * 1 + 1
    assert bench.launches_from_stats({"tier": np.array([2])}) == 2
    # top-down runs [1, 1] and [1] with 4 pairs per body entry: 2 entries x 4 pairs x 2
    assert bench.launches_from_stats(st, td_chain=4) == 1 + 2 + 2 + 2 * 4 * 2 + 3 * 1 + 1
    five = {"tier": np.array([0, 1, 1, 1, 1, 1, 0, 2])}  # one run of 5: 2 entries of 3 pairs
    assert bench.launches_from_stats(five, td_chain=3) == 1 + 2 + 2 * 3 * 2 + 1
    assert bench.launches_from_stats(five, td_chain=1) == 1 + 2 + 2 * 5 + 1
    # a tier-1 level that ran as p passes (the record's `pad`) takes p (k_explore, k_compact)
    # pairs of the chain: two levels of 3 and 2 passes = five pairs
    passes = {"tier": np.array([1, 1]), "pad": np.array([3, 2])}
    assert bench.launches_from_stats(passes, td_chain=1) == 1 + 2 * 5 + 1
    assert bench.launches_from_stats(passes, td_chain=3) == 1 + 2 * 3 * 2 + 1
    # one bottom-up run of one level, 3 triples per entry: 1 entry x 3 x 3 launches
    assert bench.launches_from_stats(st, td_chain=4, bu_chain=3) == 1 + 2 + 2 + 16 + 9 + 1
    bu4 = {"tier": np.array([1, 3, 3, 3, 3, 1, 2])}  # bottom-up run of 4: 2 entries of 3
    assert bench.launches_from_stats(bu4, td_chain=1, bu_chain=3) == 1 + 2 * 2 + 2 * 3 * 3 + 1
    # universal bodies (S C T^td C S from the entry tier on): [S S T T T S] runs in one entry
    td = {"tier": np.array([0, 0, 1, 1, 1, 0, 2])}
    assert bench.launches_from_stats(td, td_chain=4, universal=1) == 1 + (1 + 1 + 8 + 1 + 1) + 1
    # a top-down run longer than the chain re-enters at T: S C T^2 C S, then T^2 C S
    td5 = {"tier": np.array([0, 1, 1, 1, 0])}
    assert bench.launches_from_stats(td5, td_chain=2, universal=1) == 1 + 8 + 6 + 1
    # direction-optimising sequence S C T^1 B^2 T^1 C S; entry at B for a bottom-up start
    do = {"tier": np.array([1, 3, 3, 1, 4, 0])}
    assert bench.launches_from_stats(do, 1, 2, universal=1, direction=1) == 1 + (2 + 6 + 2 + 1 + 1) + 1
    # prologue: the whole sequence once after k_init (S C T^4 C S = 12 launches), then the loop
    assert bench.launches_from_stats(td, td_chain=4, universal=1, prologue=1) == 1 + 12 + 1
    assert bench.launches_from_stats(td5, td_chain=2, universal=1, prologue=1) == 1 + 8 + 6 + 1
    # a first level that is already top-down: S and C idle in the prologue
    assert bench.launches_from_stats({"tier": np.array([1, 0])}, 4, universal=1,
                                     prologue=1) == 1 + 12 + 1
    # an empty level sequence still launches the prologue
    assert bench.launches_from_stats({"tier": np.array([2])}, 4, universal=1, prologue=1) == 14

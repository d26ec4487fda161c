"""NEXT-4: one traversal over G ranks, 1-D vertex partition.

CPU (-m "not gpu"): the real driver (paper_2209_08764_b200.dist.traverse / connect) on a
world-size-2/3 gloo group, each rank a numpy stand-in with the library's per-level semantics
(tests/dist_numpy_rank.py): phase order, exchange, termination agreement and the final
combination; and the same stand-ins in one process (loopback).  GPU (-m gpu): the library's
kernels (k_explore routing candidates into the owners' receive segments, k_dist_owner /
k_dist_keep / k_dist_publish / k_dist_advance) on G handles in one process (loopback: the
peers' addresses are plain device pointers, the phases run rank by rank), levels bit-exact
with the oracle and parents valid by the certificate, plus the argument checks.
"""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import graphgen
import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from dist_numpy_rank import NumpyRank  # noqa: E402


def _graphs():
    rng = np.random.default_rng(7)
    gs = [graphgen.from_edges(60, [(i, i + 1) for i in range(59)], name="path-60"),
          graphgen.from_edges(9, [(0, 1), (0, 2), (1, 3), (2, 3), (3, 4), (5, 6)], name="small"),
          graphgen.from_edges(4, [(0, 1), (1, 2), (2, 3)], symmetrize=False, name="directed"),
          graphgen.from_edges(1, [], name="single")]
    n, m = 400, 1500
    e = np.stack([rng.integers(0, n, m), rng.integers(0, n, m)], 1)
    gs.append(graphgen.from_edges(n, e, symmetrize=False, name="rand-directed"))
    gs.append(graphgen.grid(12, 17))
    return gs


def _check(g, s, lv, pa):
    ref, _ = oracle.bfs(g.row_offsets, g.col_indices, s)
    assert np.array_equal(np.asarray(lv), ref), (g.name, s)
    code, v = oracle.check_bfs(g.row_offsets, g.col_indices, s, np.asarray(lv, dtype=np.int32),
                               np.asarray(pa, dtype=np.int32))
    assert code == 0, (g.name, s, oracle.CHECK_CODES[code], v)


def _free_port():
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def _worker(rank, world, port, out):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from dist_numpy_rank import NumpyRank as NR
    import paper_2209_08764_b200.dist as pd
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    res = {}
    for g in _graphs():
        rk = [NR(g.row_offsets, g.col_indices, rank, world)]
        pd.connect(rk, dist.group.WORLD)
        for s in sorted({0, g.n // 2, g.n - 1}):
            (lv, pa), = pd.traverse(rk, s, group=dist.group.WORLD)
            res[(g.name, s)] = (lv.tolist(), pa.tolist())
    out[rank] = res
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_protocol(world):
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    gs = {g.name: g for g in _graphs()}
    for key, (lv, pa) in res[0].items():
        g = gs[key[0]]
        _check(g, key[1], lv, pa)
        for r in range(1, world):  # every rank ends with the identical answer
            assert res[r][key] == (lv, pa), key


def test_loopback_protocol_numpy():
    sys.path.insert(0, ROOT)
    import paper_2209_08764_b200.dist as pd
    for g in _graphs():
        for G in (1, 2, 4):
            rk = [NumpyRank(g.row_offsets, g.col_indices, r, G) for r in range(G)]
            pd.connect(rk)
            for s in sorted({0, g.n - 1}):
                for lv, pa in pd.traverse(rk, s):
                    _check(g, s, lv.numpy(), pa.numpy())


# ---- GPU: the library's dist kernels -----------------------------------------------------
def _gpu_ranks(g, G, **kw):
    pkg = pytest.importorskip("paper_2209_08764_b200")
    ro = torch.from_numpy(g.row_offsets).cuda()
    col = (torch.from_numpy(g.col_indices).cuda() if g.nnz
           else torch.empty(0, dtype=torch.int32, device="cuda"))
    import paper_2209_08764_b200.dist as pd
    ranks = [pkg.DistRank(ro, col, r, G, pkg.Options(**kw)) for r in range(G)]
    pd.connect(ranks)
    return ranks


@pytest.mark.gpu
@pytest.mark.parametrize("G", [2, 3])
@pytest.mark.parametrize("kw", [dict(), dict(reorder=-1), dict(debug_poison=1, edges_per_cta=1),
                                dict(hub_vertices=1, tag_mode_pct=101),
                                dict(hub_vertices=-1, tag_mode_pct=-1)],
                         ids=["default", "no-reorder", "poison-grain1", "tags-always",
                              "bitmap-only"])
def test_gpu_loopback_small(G, kw):
    import paper_2209_08764_b200.dist as pd
    for g in _graphs():
        ranks = _gpu_ranks(g, G, **kw)
        for s in sorted({0, g.n // 2, g.n - 1}):
            outs = pd.traverse(ranks, s)
            torch.cuda.synchronize()
            for lv, pa in outs:
                _check(g, s, lv.cpu().numpy(), pa.cpu().numpy())
        for r in ranks:
            r.close()


@pytest.mark.gpu
@pytest.mark.parametrize("cfg,G,nsrc", [("rmat20", 2, 3), ("rmat20", 4, 2), ("er", 3, 4)])
def test_gpu_loopback_configs(cfg, G, nsrc):
    import paper_2209_08764_b200.dist as pd
    g = graphgen.make_config(cfg)
    ranks = _gpu_ranks(g, G)
    for s in g.sources[:nsrc]:
        outs = pd.traverse(ranks, int(s))
        torch.cuda.synchronize()
        ref = None
        for lv, pa in outs:
            lvn, pan = lv.cpu().numpy(), pa.cpu().numpy()
            _check(g, int(s), lvn, pan)
            if ref is None:
                ref = (lvn, pan)
            else:  # the combined answer is the same on every rank
                assert np.array_equal(ref[0], lvn) and np.array_equal(ref[1], pan)
    for r in ranks:
        r.close()


@pytest.mark.gpu
def test_gpu_dist_argument_checks():
    pkg = pytest.importorskip("paper_2209_08764_b200")
    import paper_2209_08764_b200.dist as pd
    g = graphgen.from_edges(3, [(0, 1), (1, 2)])
    ro = torch.from_numpy(g.row_offsets).cuda()
    col = torch.from_numpy(g.col_indices).cuda()
    lv = torch.empty(3, dtype=torch.int32, device="cuda")
    with pytest.raises(pkg.S3BFSError, match="invalid argument"):
        pkg.DistRank(ro, col, 2, 2)
    with pytest.raises(pkg.S3BFSError, match="unsupported"):
        pkg.DistRank(ro, col, 0, 2, pkg.Options(direction=1))
    with pytest.raises(pkg.S3BFSError, match="unsupported"):
        pkg.DistRank(ro, col, 0, 9)
    r0, r1 = pkg.DistRank(ro, col, 0, 2), pkg.DistRank(ro, col, 1, 2)
    with pytest.raises(pkg.S3BFSError, match="unsupported"):
        pkg.s3bfs_run(r0.handle, 0, lv, lv.clone())
    with pytest.raises(pkg.S3BFSError, match="unsupported"):
        pkg.s3bfs_clone(r0.handle)
    plain = pkg.S3BFS(ro, col)
    with pytest.raises(pkg.S3BFSError, match="unsupported"):
        pkg.s3bfs.s3bfs_dist_explore(plain.handle)
    with pytest.raises(pkg.S3BFSError, match="invalid argument"):  # one record per rank
        r0.connect([r0.export()], use_ipc=False)
    with pytest.raises(pkg.S3BFSError, match="invalid argument"):  # rank order
        r0.connect([r1.export(), r0.export()], use_ipc=False)
    pd.connect([r0, r1])
    with pytest.raises(pkg.S3BFSError, match="invalid argument"):
        r0.begin(3)
    (a, b), _ = pd.traverse([r0, r1], 0)
    _check(g, 0, a.cpu().numpy(), b.cpu().numpy())
    for x in (r0, r1, plain):
        x.close()


@pytest.mark.gpu
def test_gpu_dist_each_rank_owns_its_vertices():
    """Before the combination every rank holds exactly its own vertices' answer (block-cyclic
    32-id blocks of the internal ids; with reorder=-1 internal ids are the caller ids)."""
    pkg = pytest.importorskip("paper_2209_08764_b200")
    g = graphgen.rmat(12, 16, seed=5)
    ro = torch.from_numpy(g.row_offsets).cuda()
    col = torch.from_numpy(g.col_indices).cuda()
    import paper_2209_08764_b200.dist as pd
    G = 3
    ranks = [pkg.DistRank(ro, col, r, G, pkg.Options(reorder=-1)) for r in range(G)]
    pd.connect(ranks)
    s = int(np.argmax(np.diff(g.row_offsets)))
    for r in ranks:
        r.begin(s)
    while True:
        for r in ranks:
            r.explore()
        for r in ranks:
            r.dedup()
        if {r.advance(None)[0] for r in ranks} == {True}:
            break
    ref, _ = oracle.bfs(g.row_offsets, g.col_indices, s)
    owner = (np.arange(g.n) // 32) % G
    for r in ranks:
        lv, _ = r.end()
        lv = lv.cpu().numpy()
        mine = owner == r.rank
        assert np.array_equal(lv[mine], ref[mine])
        assert np.all(lv[~mine] == -1)
    for r in ranks:
        r.close()


@pytest.mark.gpu
@pytest.mark.parametrize("lag", [0, 1, 5])
def test_gpu_loopback_lagged_termination(lag):
    """The driver enqueues levels without a host round trip and reads each level's termination
    flag `lag` levels late; the levels enqueued past the end are no-ops on the device."""
    import paper_2209_08764_b200.dist as pd
    for g in _graphs():
        ranks = _gpu_ranks(g, 3)
        for s in sorted({0, g.n - 1}):
            for lv, pa in pd.traverse(ranks, s, lag=lag):
                _check(g, s, lv.cpu().numpy(), pa.cpu().numpy())
        for r in ranks:
            r.close()

"""NEXT-4: one traversal over G ranks, the replicated-graph edge split.

CPU (-m "not gpu"): the real driver (paper_2209_08764_b200.dist.traverse) and the real
collectives on a world-size-2/3 gloo group, each rank a numpy stand-in with the library's
per-level semantics (tests/dist_numpy_rank.py) -- the exchange protocol, padding, rank order
and termination.  GPU (-m gpu): the library's dist kernels (k_explore/k_compact on a rank's
edge slice, k_merge_min/k_merge_keep) on G handles in one process (loopback exchange), levels
bit-exact with the oracle and parents valid by the certificate, plus the argument checks.
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
        for s in sorted({0, g.n // 2, g.n - 1}):
            (lv, pa), = pd.traverse([NR(g.row_offsets, g.col_indices, rank, world)], s,
                                    group=dist.group.WORLD)
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
            for s in sorted({0, g.n - 1}):
                outs = pd.traverse([NumpyRank(g.row_offsets, g.col_indices, r, G) for r in range(G)], s)
                for lv, pa in outs:
                    _check(g, s, lv, pa)


# ---- GPU: the library's dist kernels -----------------------------------------------------
def _gpu_ranks(g, G, **kw):
    pkg = pytest.importorskip("paper_2209_08764_b200")
    ro = torch.from_numpy(g.row_offsets).cuda()
    col = (torch.from_numpy(g.col_indices).cuda() if g.nnz
           else torch.empty(0, dtype=torch.int32, device="cuda"))
    return [pkg.DistRank(ro, col, r, G, pkg.Options(**kw)) for r in range(G)]


@pytest.mark.gpu
@pytest.mark.parametrize("G", [2, 3])
@pytest.mark.parametrize("kw", [dict(), dict(reorder=-1), dict(debug_poison=1, edges_per_cta=1)],
                         ids=["default", "no-reorder", "poison-grain1"])
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
            else:  # replicated state: every rank holds the same answer
                assert np.array_equal(ref[0], lvn) and np.array_equal(ref[1], pan)
    for r in ranks:
        r.close()


@pytest.mark.gpu
def test_gpu_dist_argument_checks():
    pkg = pytest.importorskip("paper_2209_08764_b200")
    g = graphgen.from_edges(3, [(0, 1), (1, 2)])
    ro = torch.from_numpy(g.row_offsets).cuda()
    col = torch.from_numpy(g.col_indices).cuda()
    lv = torch.empty(3, dtype=torch.int32, device="cuda")
    with pytest.raises(pkg.S3BFSError, match="invalid argument"):
        pkg.DistRank(ro, col, 2, 2)
    with pytest.raises(pkg.S3BFSError, match="unsupported"):
        pkg.DistRank(ro, col, 0, 2, pkg.Options(direction=1))
    r = pkg.DistRank(ro, col, 0, 2)
    with pytest.raises(pkg.S3BFSError, match="unsupported"):
        pkg.s3bfs_run(r.handle, 0, lv, lv.clone())
    plain = pkg.S3BFS(ro, col)
    with pytest.raises(pkg.S3BFSError, match="unsupported"):
        pkg.s3bfs.s3bfs_dist_expand(plain.handle)
    with pytest.raises(pkg.S3BFSError, match="invalid argument"):
        r.begin(3)
    r.begin(0)
    n_local, done = r.expand()
    assert not done
    with pytest.raises(pkg.S3BFSError, match="invalid argument"):  # count > stride
        r.merge(torch.zeros((1, 4), dtype=torch.int32, device="cuda"), [2, 0], 1)
    r.close()
    plain.close()


@pytest.mark.gpu
def test_gpu_dist_clone():
    """A clone of a dist handle (shared prepared graph, own workspace) runs the protocol too."""
    pkg = pytest.importorskip("paper_2209_08764_b200")
    import paper_2209_08764_b200.dist as pd
    g = _graphs()[4]  # rand-directed
    ranks = _gpu_ranks(g, 2)
    clones = []
    for r in ranks:
        c = pd.DistRank.__new__(pd.DistRank)
        c.rank, c.size, c.n, c.device, c.stream = r.rank, r.size, r.n, r.device, None
        c.row_offsets, c.col_indices = r.row_offsets, r.col_indices
        c.handle = pkg.s3bfs_clone(r.handle)
        c.level, c.parent = torch.empty_like(r.level), torch.empty_like(r.parent)
        clones.append(c)
    for s in (0, g.n - 1):
        for lv, pa in pd.traverse(clones, s):
            _check(g, s, lv.cpu().numpy(), pa.cpu().numpy())
    for c in clones + ranks:
        c.close()

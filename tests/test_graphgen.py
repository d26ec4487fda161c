"""Seeded input generator: determinism, CSR invariants and the config recipes (CPU only)."""
import hashlib

import numpy as np
import pytest

import graphgen


def digest(g):
    return hashlib.sha256(g.row_offsets.tobytes() + g.col_indices.tobytes()).hexdigest()


def check_csr(g, simple=True, symmetric=True):
    ro, col = g.row_offsets, g.col_indices
    assert ro[0] == 0 and ro[-1] == col.size
    assert np.all(np.diff(ro) >= 0)
    assert col.size == 0 or (col.min() >= 0 and col.max() < g.n)
    src = np.repeat(np.arange(g.n, dtype=np.int64), np.diff(ro))
    if simple:
        assert not np.any(src == col)                              # no self-loops
        key = src * g.n + col
        assert np.all(np.diff(key) > 0)                            # sorted rows, no duplicates
    if symmetric:
        fwd = np.sort(src * g.n + col)
        bwd = np.sort(col.astype(np.int64) * g.n + src)
        assert np.array_equal(fwd, bwd)


def test_from_edges_spec_examples():
    g = graphgen.from_edges(3, [(0, 1), (1, 2)], symmetrize=False)
    assert g.row_offsets.tolist() == [0, 1, 2, 2] and g.col_indices.tolist() == [1, 2]
    g = graphgen.from_edges(4, [], symmetrize=False)
    assert g.row_offsets.tolist() == [0, 0, 0, 0, 0] and g.nnz == 0
    g = graphgen.from_edges(2, [(0, 1)], symmetrize=True)
    assert g.row_offsets.tolist() == [0, 1, 2] and g.col_indices.tolist() == [1, 0]
    g = graphgen.from_edges(3, [(0, 1), (0, 1), (1, 1)], symmetrize=False)  # multigraph kept
    assert g.col_indices.tolist() == [1, 1, 1]
    with pytest.raises(RuntimeError):
        graphgen.from_edges(2, [(0, 5)])


def test_grid_exact_counts():
    g = graphgen.grid(1024, 1024)
    assert g.n == 1 << 20 and g.nnz == 4_190_208 and g.nnz // 2 == 2_095_104
    check_csr(g)
    deg = g.degrees()
    assert deg.min() == 2 and deg.max() == 4 and (deg == 2).sum() == 4


def test_er_config_and_determinism():
    g1 = graphgen.make_config("er")
    g2 = graphgen.make_config("er")
    assert digest(g1) == digest(g2) and g1.sources == g2.sources
    check_csr(g1)
    assert g1.n == 1 << 16 and g1.nnz // 2 <= 1 << 19 and g1.nnz // 2 > (1 << 19) - 200
    assert len(set(g1.sources)) == 8
    g3 = graphgen.er(1 << 16, 1 << 19, seed=2)
    assert digest(g3) != digest(g1)
    # thread count does not change the output (counter-based draws)
    assert digest(graphgen.er(1 << 12, 1 << 15, seed=3, threads=1)) == \
        digest(graphgen.er(1 << 12, 1 << 15, seed=3, threads=7))


def test_rmat_determinism_and_quadrants():
    a = graphgen.rmat(14, 16, seed=5, threads=1)
    b = graphgen.rmat(14, 16, seed=5, threads=5)
    assert digest(a) == digest(b)
    check_csr(a)
    # before permutation the top id bit is 0 for the source with probability a+b = 0.76:
    # in the symmetrised graph the fraction of arcs with both endpoints in the low half is
    # ~a/(1-d-...) -- use the direct statistic on the unpermuted graph instead:
    u = graphgen.rmat(16, 16, seed=11, permute=False)
    src = np.repeat(np.arange(u.n), u.degrees())
    col = u.col_indices
    half = u.n // 2
    low_low = np.mean((src < half) & (col < half))
    hi_hi = np.mean((src >= half) & (col >= half))
    # symmetrised quadrant masses (before dedup): a = 0.57 in low/low, d = 0.05 in high/high
    assert 0.45 < low_low < 0.60 and 0.03 < hi_hi < 0.07


def test_rmat20_config_shape():
    g = graphgen.make_config("rmat20")
    check_csr(g)
    deg = g.degrees()
    assert g.n == 1 << 20 and 30_000_000 < g.nnz < 32_500_000
    assert 0.30 < (deg == 0).mean() < 0.45
    assert len(set(g.sources)) == 16 and all(deg[s] > 0 for s in g.sources)


def test_tail_small_recipe():
    g = graphgen.rmat_tail(scale=12, ef=16, seed=4, path_len=500)
    check_csr(g)
    m = g.meta
    assert g.n == (1 << 12) + 500 and m["path_first"] == 1 << 12 and m["far_end"] == g.n - 1
    deg = g.degrees()
    assert deg[m["far_end"]] == 1 and np.all(deg[m["path_first"] + 1:m["far_end"]] == 2)
    assert m["anchor"] in g.col_indices[g.row_offsets[m["path_first"]]:g.row_offsets[m["path_first"] + 1]]

"""Pins for the CPU oracle (oracle/) against things other than itself (CPU only).

Each oracle function is checked against brute force, closed forms, invariants or the
worked examples in tests/golden/spec_examples.json -- chosen so that a dropped term, a
wrong sign/index or a transposed operand in the oracle fails at least one of them.
"""
import itertools
import json
import os

import numpy as np
import pytest

import graphgen
import oracle

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))
INF = 1 << 40


def brute_levels(n, arcs, s):
    """Unit-weight Floyd-Warshall over the arc list (no CSR, no queue): dist[s][.] or -1."""
    D = np.full((n, n), INF, dtype=np.int64)
    np.fill_diagonal(D, 0)
    for u, v in arcs:
        if u != v:
            D[u, v] = min(D[u, v], 1)
    for k in range(n):
        D = np.minimum(D, D[:, k:k + 1] + D[k:k + 1, :])
    row = D[s]
    return np.where(row >= INF, -1, row).astype(np.int32)


def csr(n, arcs, directed=True):
    return graphgen.from_edges(n, arcs, symmetrize=not directed, dedup=False,
                               drop_self_loops=False)


def arcs_of(g):
    ro, col = g.row_offsets, g.col_indices
    return [(u, int(col[k])) for u in range(g.n) for k in range(ro[u], ro[u + 1])]


# ---------------------------------------------------------------------------------------
# oracle_bfs vs brute force
# ---------------------------------------------------------------------------------------
def test_bfs_all_undirected_graphs_up_to_5_vertices():
    for n in range(1, 6):
        pairs = list(itertools.combinations(range(n), 2))
        for mask in range(1 << len(pairs)):
            edges = [pairs[i] for i in range(len(pairs)) if mask >> i & 1]
            g = csr(n, edges, directed=False)
            arcs = arcs_of(g)
            for s in range(n):
                level, parent = oracle.bfs(g.row_offsets, g.col_indices, s)
                assert np.array_equal(level, brute_levels(n, arcs, s)), (n, edges, s)
                assert oracle.check_bfs(g.row_offsets, g.col_indices, s, level, parent)[0] == 0


def test_bfs_all_directed_graphs_on_3_vertices_with_self_loops():
    arcs_all = [(u, v) for u in range(3) for v in range(3)]
    for mask in range(1 << len(arcs_all)):
        arcs = [arcs_all[i] for i in range(len(arcs_all)) if mask >> i & 1]
        g = csr(3, arcs)
        for s in range(3):
            level, parent = oracle.bfs(g.row_offsets, g.col_indices, s)
            assert np.array_equal(level, brute_levels(3, arcs, s))
            assert oracle.check_bfs(g.row_offsets, g.col_indices, s, level, parent)[0] == 0


@pytest.mark.parametrize("seed", range(12))
def test_bfs_random_multigraphs_vs_brute_force(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(2, 80))
    m = int(rng.integers(0, 4 * n))
    arcs = [(int(a), int(b)) for a, b in rng.integers(0, n, size=(m, 2))]
    arcs += arcs[: m // 5]                      # duplicate arcs (multigraph, reading R14)
    g = csr(n, arcs, directed=bool(seed % 2))
    garcs = arcs_of(g)
    for s in rng.choice(n, size=min(n, 6), replace=False):
        level, parent = oracle.bfs(g.row_offsets, g.col_indices, int(s))
        assert np.array_equal(level, brute_levels(n, garcs, int(s)))
        assert oracle.check_bfs(g.row_offsets, g.col_indices, int(s), level, parent)[0] == 0


def test_bfs_spec_examples():
    for ex in GOLDEN["serial_bfs"]:
        g = csr(ex["n"], ex["edges"], directed=False)
        level, _ = oracle.bfs(g.row_offsets, g.col_indices, ex["source"])
        assert level.tolist() == ex["level"], ex["cite"]


def test_bfs_rejects_bad_source():
    g = csr(3, [(0, 1)])
    with pytest.raises(oracle.OracleError):
        oracle.bfs(g.row_offsets, g.col_indices, 3)
    with pytest.raises(oracle.OracleError):
        oracle.bfs(g.row_offsets, g.col_indices, -1)


# closed forms ---------------------------------------------------------------------------
@pytest.mark.parametrize("R,C,src", [(7, 9, (0, 0)), (7, 9, (3, 4)), (1, 13, (0, 5)), (16, 16, (15, 0))])
def test_bfs_grid_is_manhattan(R, C, src):
    g = graphgen.grid(R, C)
    s = src[0] * C + src[1]
    level, _ = oracle.bfs(g.row_offsets, g.col_indices, s)
    r, c = np.divmod(np.arange(R * C), C)
    assert np.array_equal(level, np.abs(r - src[0]) + np.abs(c - src[1]))


def test_bfs_full_grid_config_closed_form():
    g = graphgen.grid(1024, 1024)
    r, c = np.divmod(np.arange(g.n), 1024)
    for s in (0, 512 * 1024 + 512):
        level, _ = oracle.bfs(g.row_offsets, g.col_indices, s)
        assert np.array_equal(level, np.abs(r - s // 1024) + np.abs(c - s % 1024))
    assert level.max() == 1024  # eccentricity of the centre (reading R21)


@pytest.mark.parametrize("n", [1, 2, 5, 64])
def test_bfs_cycle_path_star_complete(n):
    i = np.arange(n)
    cyc = csr(n, [(k, (k + 1) % n) for k in range(n)] if n > 1 else [], directed=False)
    path = csr(n, [(k, k + 1) for k in range(n - 1)], directed=False)
    star = csr(n, [(0, k) for k in range(1, n)], directed=False)
    comp = csr(n, [(a, b) for a in range(n) for b in range(a + 1, n)], directed=False)
    for s in {0, n // 2, n - 1}:
        assert np.array_equal(oracle.bfs(cyc.row_offsets, cyc.col_indices, s)[0],
                              np.minimum(np.abs(i - s), n - np.abs(i - s)))
        assert np.array_equal(oracle.bfs(path.row_offsets, path.col_indices, s)[0], np.abs(i - s))
        lv = oracle.bfs(star.row_offsets, star.col_indices, s)[0]
        exp = np.where(i == s, 0, np.where((i == 0) | (s == 0), 1, 2))
        assert np.array_equal(lv, exp)
        assert np.array_equal(oracle.bfs(comp.row_offsets, comp.col_indices, s)[0],
                              (i != s).astype(np.int32))


def test_bfs_binary_tree_depth():
    n = 2 ** 10 - 1
    g = csr(n, [(k, 2 * k + 1) for k in range(n) if 2 * k + 1 < n] +
            [(k, 2 * k + 2) for k in range(n) if 2 * k + 2 < n], directed=False)
    level, _ = oracle.bfs(g.row_offsets, g.col_indices, 0)
    assert np.array_equal(level, np.floor(np.log2(np.arange(n) + 1)).astype(np.int32))


# ---------------------------------------------------------------------------------------
# certificate: mutation tests (each corruption must be caught and name the vertex)
# ---------------------------------------------------------------------------------------
def test_certificate_catches_mutations():
    g = graphgen.grid(9, 11)
    ro, col = g.row_offsets, g.col_indices
    s = 40
    level, parent = oracle.bfs(ro, col, s)
    assert oracle.check_bfs(ro, col, s, level, parent) == (0, -1)
    v = 77
    # level +1 / -1
    for d in (+1, -1):
        lv = level.copy(); lv[v] += d
        code, bad = oracle.check_bfs(ro, col, s, lv, parent)
        assert code != 0 and bad >= 0
    # reachable vertex marked unreachable
    lv = level.copy(); pa = parent.copy(); lv[v] = -1; pa[v] = -1
    code, bad = oracle.check_bfs(ro, col, s, lv, pa)
    assert code in (3, 5) and (bad == v or parent[bad] == v)   # v itself or a child of v
    # parent replaced by a non-neighbour at the right level
    pa = parent.copy()
    cands = [u for u in range(g.n) if level[u] == level[v] - 1 and u not in col[ro[v]:ro[v + 1]]]
    pa[v] = cands[0]
    assert oracle.check_bfs(ro, col, s, level, pa) == (4, v)
    # parent replaced by a same-level vertex
    pa = parent.copy(); pa[v] = [u for u in range(g.n) if level[u] == level[v] and u != v][0]
    assert oracle.check_bfs(ro, col, s, level, pa) == (3, v)
    # parent[s] != s
    pa = parent.copy(); pa[s] = col[ro[s]]
    assert oracle.check_bfs(ro, col, s, level, pa) == (1, s)
    # unreachable vertex given a level (two components)
    g2 = csr(4, [(0, 1), (2, 3)], directed=False)
    lv, pa = oracle.bfs(g2.row_offsets, g2.col_indices, 0)
    lv2 = lv.copy(); lv2[2] = 1
    assert oracle.check_bfs(g2.row_offsets, g2.col_indices, 0, lv2, pa)[0] != 0
    pa2 = pa.copy(); pa2[3] = 2
    assert oracle.check_bfs(g2.row_offsets, g2.col_indices, 0, lv, pa2) == (6, 3)


# ---------------------------------------------------------------------------------------
# scans (Fig.1 L14-L15)
# ---------------------------------------------------------------------------------------
def test_scan_spec_examples():
    for ex in GOLDEN["inclusive_scan"]:
        assert oracle.inclusive_scan(ex["in"]).tolist() == ex["out"], ex["cite"]


@pytest.mark.parametrize("n", [0, 1, 2, 31, 32, 33, 1000, 4097])
def test_scan_closed_forms(n):
    i = np.arange(n, dtype=np.int64)
    assert np.array_equal(oracle.exclusive_scan(np.ones(n, np.int32)), np.arange(n + 1))
    assert np.array_equal(oracle.exclusive_scan(i.astype(np.int32)),
                          np.arange(n + 1) * (np.arange(n + 1) - 1) // 2)
    assert np.array_equal(oracle.inclusive_scan(np.full(n, 3, np.int32)), 3 * (i + 1))
    assert oracle.exclusive_scan(np.zeros(n, np.int32)).tolist() == [0] * (n + 1)


def test_scan_vs_numpy_cumsum_and_overflow():
    rng = np.random.default_rng(5)
    for _ in range(20):
        a = rng.integers(0, 1000, size=int(rng.integers(0, 100000))).astype(np.int32)
        ex = oracle.exclusive_scan(a)
        assert ex[0] == 0 and np.array_equal(ex[1:], np.cumsum(a, dtype=np.int64))
        assert np.array_equal(oracle.inclusive_scan(a), np.cumsum(a, dtype=np.int64))
    big = np.full(3, 2 ** 30, np.int32)
    with pytest.raises(oracle.OracleError):
        oracle.exclusive_scan(big)


# ---------------------------------------------------------------------------------------
# Find-StartExpPoint (range rule) vs brute force linear search
# ---------------------------------------------------------------------------------------
def test_start_points_spec_examples():
    for ex in GOLDEN["find_start_points"]:
        u, off = oracle.find_start_points(ex["edge_sum"], ex["chunk"], ex["p_l"])
        assert u.tolist() == ex["u"] and off.tolist() == ex["off"], ex["cite"]


@pytest.mark.parametrize("seed", range(20))
def test_start_points_vs_linear_search(seed):
    rng = np.random.default_rng(seed)
    n_l = int(rng.integers(1, 300))
    deg = rng.integers(0, 12, size=n_l) * (rng.random(n_l) < 0.7)
    deg[rng.integers(0, n_l)] += 1                   # e_l >= 1
    incl = np.cumsum(deg)
    e_l = int(incl[-1])
    p_l = int(rng.integers(1, e_l + 1))
    chunk = -(-e_l // p_l)
    p_used = -(-e_l // chunk)                          # workers whose start is < e_l
    u, off = oracle.find_start_points(incl.astype(np.int32), chunk, p_l)
    excl = np.concatenate([[0], incl[:-1]])
    for t in range(p_l):
        st = t * chunk
        if t >= p_used:
            assert u[t] == -1
            continue
        uu = next(k for k in range(n_l) if excl[k] <= st < incl[k])   # linear search
        assert (u[t], off[t]) == (uu, st - excl[uu])
        assert 0 <= off[t] < deg[u[t]]


# ---------------------------------------------------------------------------------------
# Dedup + linearise (Fig.1 L19-L29)
# ---------------------------------------------------------------------------------------
def test_dedup_linearize_spec_and_trivial():
    ex = GOLDEN["dedup_linearize"][0]
    owner = np.zeros(10, np.int32)
    for k, w in ex["owner"].items():
        owner[int(k)] = w
    sizes, fr = oracle.dedup_linearize(ex["queues"], owner)
    assert sizes.tolist() == ex["sizes"] and fr.tolist() == ex["frontier"], ex["cite"]
    sizes, fr = oracle.dedup_linearize([[], [], []], owner)            # all empty
    assert sizes.tolist() == [0, 0, 0] and fr.tolist() == []
    sizes, fr = oracle.dedup_linearize([[3, 1, 2]], np.zeros(4, np.int32))  # single worker
    assert sizes.tolist() == [3] and fr.tolist() == [3, 1, 2]


# ---------------------------------------------------------------------------------------
# Figure 1 end to end: levels vs brute force; stats vs SPEC examples and direct counts
# ---------------------------------------------------------------------------------------
def test_fig1_spec_stats():
    for ex in GOLDEN["run_bfs_stats"]:
        if "star_leaves" in ex:
            k = ex["star_leaves"]
            g = csr(k + 1, [(0, j) for j in range(1, k + 1)], directed=True)
        else:
            g = csr(ex["n"], ex["edges"], directed=ex["directed"])
        _, nl, el, pl = oracle.s3bfs_fig1(g.row_offsets, g.col_indices, ex["source"], ex["P"])
        assert nl.tolist() == ex["n_l"] and el.tolist() == ex["e_l"] and pl.tolist() == ex["p_l"], ex["cite"]


@pytest.mark.parametrize("seed", range(10))
def test_fig1_levels_and_accounting(seed):
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(2, 70))
    arcs = [(int(a), int(b)) for a, b in rng.integers(0, n, size=(int(rng.integers(0, 3 * n)), 2))]
    g = csr(n, arcs, directed=bool(seed % 2))
    garcs = arcs_of(g)
    deg = np.diff(g.row_offsets)
    for s in rng.choice(n, size=min(n, 4), replace=False):
        exp = brute_levels(n, garcs, int(s))
        for P in (1, 2, 3, 4, 8, 16):
            level, nl, el, pl = oracle.s3bfs_fig1(g.row_offsets, g.col_indices, int(s), P)
            assert np.array_equal(level, exp), (seed, s, P)
            L = exp.max() + 1
            assert nl.tolist() == [int((exp == l).sum()) for l in range(L)]
            assert el.tolist() == [int(deg[exp == l].sum()) for l in range(L)]
            assert pl.tolist() == [min(P, e) for e in el.tolist()]
            assert el.sum() == sum(1 for (u, _) in garcs if exp[u] >= 0)   # P:41 accounting


def _grid_corner_profile(R, C):
    """Closed form for a 4-neighbour R x C grid BFS'd from corner (0,0) (level = r + c):
    n_l = min(l, R-1, C-1, R+C-2-l) + 1 (anti-diagonal length), and e_l = 4 n_l minus one
    missing neighbour per border side the diagonal touches -- no level array involved."""
    L = R + C - 1
    nl = [min(l, R - 1, C - 1, R + C - 2 - l) + 1 for l in range(L)]
    el = [4 * nl[l] - (l <= C - 1) - (R - 1 <= l) - (l <= R - 1) - (C - 1 <= l) for l in range(L)]
    return nl, el


@pytest.mark.parametrize("R,C", [(1024, 1024), (7, 3), (3, 7), (1, 9), (2, 2)])
def test_level_profile_grid_corner_closed_form(R, C):
    """oracle_level_profile's n_l / e_l (Fig1 L9, L15) and m_c pinned to
    the grid's closed forms; a rectangular grid catches a transposed r/c, the 1024^2 case is
    BASELINE configs[1] (n_l = l+1 up to 1023, then 2047-l; max e_l 4,092)."""
    g = graphgen.grid(R, C)
    level, _ = oracle.bfs(g.row_offsets, g.col_indices, 0)
    nl, el, mc, nc = oracle.level_profile(g.row_offsets, level)
    exp_nl, exp_el = _grid_corner_profile(R, C)
    assert nl.tolist() == exp_nl
    assert el.tolist() == exp_el
    # P:41 accounting: the grid is connected, so every arc of the CSR is in the component
    assert mc == g.nnz == 2 * (R * (C - 1) + C * (R - 1)) and nc == R * C
    if (R, C) == (1024, 1024):
        assert max(el) == 4092 and nl[1023] == 1024 and nl[2046] == 1


def test_level_profile_grid_centre_closed_form():
    """From the centre (512, 512) of the 1024^2 grid (BASELINE configs[1], R21): the L1 ball
    stays interior up to l = 510, so n_l = 4l and e_l = 16 l; at l = 511 it is still whole
    but (1023, 512) and (512, 1023) sit on the border (e = 16*511 - 2); the whole profile
    sums to n and to the arc count of the grid."""
    g = graphgen.grid(1024, 1024)
    level, _ = oracle.bfs(g.row_offsets, g.col_indices, 524_800)
    nl, el, mc, nc = oracle.level_profile(g.row_offsets, level)
    assert len(nl) == 1025 and nl[0] == 1 and el[0] == 4
    for l in range(1, 511):
        assert nl[l] == 4 * l and el[l] == 16 * l, l
    assert nl[511] == 4 * 511 and el[511] == 16 * 511 - 2
    assert nl.sum() == nc == 1 << 20
    assert el.sum() == mc == 4_190_208 == g.nnz


def test_level_profile_spec_examples():
    """SPEC S:274 (directed path: n_l [1,1,1,1], e_l [1,1,1,0]) and S:275 (star with 100
    leaves: n_l [1,100], e_l [100,0]) -- the out-degree sums of Fig1 L13/L15.  A profile that
    summed in-degrees (or shifted the level by one) gives [0,1,1,1] / [0,100] and fails."""
    for ex in GOLDEN["run_bfs_stats"]:
        if "star_leaves" in ex:
            k = ex["star_leaves"]
            g = csr(k + 1, [(0, j) for j in range(1, k + 1)], directed=True)
        else:
            g = csr(ex["n"], ex["edges"], directed=ex["directed"])
        level, _ = oracle.bfs(g.row_offsets, g.col_indices, ex["source"])
        nl, el, mc, nc = oracle.level_profile(g.row_offsets, level)
        assert nl.tolist() == ex["n_l"] and el.tolist() == ex["e_l"], ex["cite"]
        assert mc == sum(ex["e_l"]) == g.nnz and nc == sum(ex["n_l"]), ex["cite"]


def test_level_profile_two_components_and_unreached():
    """Unreached vertices (-1) contribute to nothing: a path 0-1-2 plus a disjoint K4 on
    3..6 from source 0 gives n_l [1,1,1], e_l [1,2,1] (undirected path degrees), m_c = 4 arcs
    of the path only (P:41 counts the source's component), n_c = 3."""
    edges = [(0, 1), (1, 2)] + [(a, b) for a in range(3, 7) for b in range(a + 1, 7)]
    g = csr(7, edges, directed=False)
    level, _ = oracle.bfs(g.row_offsets, g.col_indices, 0)
    nl, el, mc, nc = oracle.level_profile(g.row_offsets, level)
    assert nl.tolist() == [1, 1, 1] and el.tolist() == [1, 2, 1] and mc == 4 and nc == 3


def test_level_profile_vs_direct_counts():
    g = graphgen.rmat(10, 8, seed=9)
    s = int(np.argmax(np.diff(g.row_offsets)))
    level, _ = oracle.bfs(g.row_offsets, g.col_indices, s)
    nl, el, mc, nc = oracle.level_profile(g.row_offsets, level)
    deg = np.diff(g.row_offsets)
    assert nl.tolist() == np.bincount(level[level >= 0]).tolist()
    assert el.tolist() == np.bincount(level[level >= 0], weights=deg[level >= 0]).astype(int).tolist()
    assert mc == int(deg[level >= 0].sum()) and nc == int((level >= 0).sum())

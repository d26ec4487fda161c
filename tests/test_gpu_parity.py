"""GPU parity: the CUDA path through the C ABI vs the CPU oracle (oracle/, pinned separately).

Levels are compared bit-exactly (integer work); parents are validated by the certificate
(non-unique, DESIGN R2/R16); per-level n_l / e_l from the library's stats are compared with
the oracle's level profile (unique).  Every graph runs under several tier / loop settings
so that tier 0 (single CTA), tier 1 (k_explore + k_compact) and the transitions are all hit.
"""
import numpy as np
import pytest

import graphgen
import oracle

torch = pytest.importorskip("torch")
pkg = pytest.importorskip("paper_2209_08764_b200")

pytestmark = pytest.mark.gpu

# (name, options) -- debug_poison fills Owner with slot-like garbage first (DESIGN R3)
SETTINGS = [
    ("graph-default", dict(debug_poison=1)),
    ("graph-tier1-only", dict(debug_poison=1, tier0_max_edges=-1)),
    ("graph-T0=64", dict(debug_poison=1, tier0_max_edges=64)),
    ("graph-grain1", dict(debug_poison=1, tier0_max_edges=-1, edges_per_cta=1)),
    ("graph-3ctas", dict(debug_poison=1, tier0_max_edges=-1, max_ctas=3, edges_per_cta=64)),
    ("host-loop", dict(debug_poison=1, loop_mode=2, tier0_max_edges=512)),
    ("work-insensitive", dict(debug_poison=1, variant=1)),
    ("grain-4096-T0-1", dict(debug_poison=1, tier0_max_edges=1, edges_per_cta=4096)),
    # cluster tier (one 8-CTA cluster, consecutive levels): nearly every mid-size level / off
    ("cluster-T0-16", dict(debug_poison=1, tier0_max_edges=16)),
    ("cluster-only-host", dict(debug_poison=1, tier0_max_edges=-1, loop_mode=2)),
    ("no-cluster", dict(debug_poison=1, cluster_max_edges=-1)),
    ("no-reorder", dict(debug_poison=1, reorder=-1, tier0_max_edges=64)),
    # NEXT-3 direction optimisation: bottom-up on every level / switching back and forth
    ("bu-always", dict(debug_poison=1, tier0_max_edges=-1, direction=1, do_alpha=1 << 30,
                       do_beta=-1)),
    ("bu-mixed", dict(debug_poison=1, tier0_max_edges=16, direction=1, do_alpha=64, do_beta=3)),
    ("bu-no-reorder", dict(debug_poison=1, reorder=-1, tier0_max_edges=-1, direction=1,
                           do_alpha=1 << 30, do_beta=-1)),
    # k_explore's tag mode (ids >= hub_vertices tested by their discovery tag alone): tiny
    # graphs are below the default 2^20 hub ids, so these force it -- on every level, on a mix
    # of levels (50 %), after tier-0 / cluster / bottom-up levels (tags written by every tier)
    ("tags-hub1-tier1", dict(debug_poison=1, hub_vertices=1, tag_mode_pct=101,
                             tier0_max_edges=-1)),
    ("tags-hub5-T0-16", dict(debug_poison=1, hub_vertices=5, tag_mode_pct=101,
                             tier0_max_edges=16)),
    ("tags-hub3-mixed-levels", dict(debug_poison=1, hub_vertices=3, tag_mode_pct=50,
                                    tier0_max_edges=-1)),
    ("tags-hub3-bu-mixed", dict(debug_poison=1, hub_vertices=3, tag_mode_pct=101,
                                tier0_max_edges=16, direction=1, do_alpha=64, do_beta=3)),
    ("tags-never", dict(debug_poison=1, tag_mode_pct=-1, tier0_max_edges=-1)),
    # level passes (a tier-1 level in tag mode explored as consecutive edge ranges, each a
    # complete explore + dedup appending to the next frontier): forced on every tier-1 level --
    # two passes with a 1 % / 50 % first pass, five passes, with the small tiers and with the
    # host loop, and next to bottom-up levels
    ("passes-2-tier1", dict(debug_poison=1, tag_mode_pct=101, hub_vertices=3, tier0_max_edges=-1,
                            cluster_max_edges=-1, split_min_edges=1, split_first_pct=1,
                            split_passes=2)),
    ("passes-2-half-grain1", dict(debug_poison=1, tag_mode_pct=101, tier0_max_edges=-1,
                                  cluster_max_edges=-1, edges_per_cta=1, split_min_edges=1,
                                  split_first_pct=50, split_passes=2)),
    ("passes-5-T0-16", dict(debug_poison=1, tag_mode_pct=101, hub_vertices=5, tier0_max_edges=16,
                            split_min_edges=2, split_first_pct=12, split_passes=5)),
    ("passes-3-host-loop", dict(debug_poison=1, tag_mode_pct=101, loop_mode=2,
                                tier0_max_edges=64, split_min_edges=8, split_first_pct=30,
                                split_passes=3)),
    ("passes-2-bu-mixed", dict(debug_poison=1, tag_mode_pct=101, hub_vertices=3,
                               tier0_max_edges=16, direction=1, do_alpha=64, do_beta=3,
                               split_min_edges=4, split_first_pct=25, split_passes=2)),
    ("passes-off", dict(debug_poison=1, split_passes=1)),
]


def to_dev(g):
    ro = torch.from_numpy(g.row_offsets).cuda()
    col = torch.from_numpy(g.col_indices).cuda() if g.nnz else torch.empty(0, dtype=torch.int32,
                                                                           device="cuda")
    return ro, col


def check_traversal(g, bfs, s, stats=True):
    level, parent = bfs.run(s)
    torch.cuda.synchronize()
    lv, pa = level.cpu().numpy(), parent.cpu().numpy()
    ref, _ = oracle.bfs(g.row_offsets, g.col_indices, s)
    if not np.array_equal(lv, ref):
        bad = np.flatnonzero(lv != ref)
        raise AssertionError(f"{g.name} src {s}: {bad.size} levels differ, first v={bad[0]} "
                             f"gpu={lv[bad[0]]} oracle={ref[bad[0]]}")
    code, badv = oracle.check_bfs(g.row_offsets, g.col_indices, s, lv, pa)
    assert code == 0, f"{g.name} src {s}: {oracle.CHECK_CODES[code]} at v={badv}"
    if stats:
        st = bfs.level_stats()
        nl, el, _, _ = oracle.level_profile(g.row_offsets, ref)
        assert st["level"].tolist() == list(range(len(nl))), (g.name, s)
        assert np.array_equal(st["n_l"], nl), (g.name, s, st["n_l"][:10], nl[:10])
        assert np.array_equal(st["e_l"], el), (g.name, s)
        assert np.array_equal(st["kept"][:-1], nl[1:]) and st["kept"][-1] == 0
        assert np.all(st["candidates"][st["e_l"] > 0] >= st["kept"][st["e_l"] > 0])
    return lv, pa


def tiny_graphs():
    gs = []
    add = lambda name, n, e, sym=True: gs.append(  # noqa: E731
        (name, graphgen.from_edges(n, e, symmetrize=sym, name=name)))
    add("single-vertex", 1, [])
    add("single-edge", 2, [(0, 1)])
    add("path-50", 50, [(i, i + 1) for i in range(49)])
    add("path-directed", 4, [(0, 1), (1, 2), (2, 3)], sym=False)
    add("star-10000", 10001, [(0, i) for i in range(1, 10001)])   # hub row > one 4096 tile
    add("cycle-101", 101, [(i, (i + 1) % 101) for i in range(101)])
    add("complete-40", 40, [(i, j) for i in range(40) for j in range(i + 1, 40)])
    add("binary-tree-1023", 1023, [((i - 1) // 2, i) for i in range(1, 1023)])
    add("two-components", 5, [(0, 1), (1, 2), (3, 4)])
    add("isolated", 6, [(1, 2), (2, 3)])
    add("multigraph", 6, [(0, 1), (0, 1), (1, 1), (1, 2), (2, 2), (2, 3), (3, 4), (3, 4), (5, 5)])
    add("diamond", 4, [(0, 1), (0, 2), (1, 3), (2, 3)], sym=False)
    # star of stars: 300 hubs all pointing at the same 50 shared vertices (heavy duplicates)
    e = [(0, h) for h in range(1, 301)] + [(h, 301 + k) for h in range(1, 301) for k in range(50)]
    add("star-of-stars", 351, e)
    # sinks in the frontier: hub -> 20000 vertices, every 7th has one out-arc (C9)
    e = [(0, i) for i in range(1, 20001)] + [(i, 20001 + i // 7) for i in range(1, 20001, 7)]
    add("sinks-directed", 20001 + 20000 // 7 + 1, e, sym=False)
    # e_l crosses T0 up and back down: path -> broom of 9000 leaves -> path
    e = [(i, i + 1) for i in range(20)] + [(20, 21 + k) for k in range(9000)] + \
        [(21 + k, 9021) for k in range(0, 9000, 3000)] + [(9021 + i, 9022 + i) for i in range(30)]
    add("crossing", 9052, e)
    return gs


TINY = tiny_graphs()


@pytest.mark.parametrize("setting", SETTINGS, ids=[s[0] for s in SETTINGS])
def test_tiny_suite_all_sources(setting):
    _, kw = setting
    for name, g in TINY:
        ro, col = to_dev(g)
        bfs = pkg.S3BFS(ro, col, pkg.Options(**kw))
        srcs = range(g.n) if g.n <= 64 else sorted({0, 1, g.n // 2, g.n - 1})
        for s in srcs:
            check_traversal(g, bfs, s)
        bfs.close()


@pytest.mark.parametrize("seed", range(8))
def test_random_multigraphs(seed):
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(100, 30000))
    m = int(rng.integers(n // 2, 12 * n))
    # skewed endpoints (R-MAT-like hot vertices), duplicates and self-loops kept
    hot = rng.integers(0, n, size=max(1, n // 100))
    src = np.where(rng.random(m) < 0.3, rng.choice(hot, m), rng.integers(0, n, m))
    dst = rng.integers(0, n, m)
    g = graphgen.from_edges(n, np.stack([src, dst], 1), symmetrize=bool(seed % 2),
                            name=f"rand{seed}")
    ro, col = to_dev(g)
    for _, kw in SETTINGS[:5] + SETTINGS[-5:]:
        bfs = pkg.S3BFS(ro, col, pkg.Options(**kw))
        for s in rng.choice(n, 3, replace=False):
            check_traversal(g, bfs, int(s))
        bfs.close()


def test_race_confinement_repeated_runs():
    """>= 50 runs: identical levels, valid parents, duplicate-free frontiers."""
    name, g = [t for t in TINY if t[0] == "star-of-stars"][0]
    gr = graphgen.rmat(14, 16, seed=9)
    gr.name = "rmat14"
    for gg in (g, gr):
        ro, col = to_dev(gg)
        for kw in (dict(debug_poison=1), dict(debug_poison=1, tier0_max_edges=-1,
                                              edges_per_cta=16)):
            bfs = pkg.S3BFS(ro, col, pkg.Options(**kw))
            first = None
            for _ in range(50):
                lv, _ = check_traversal(gg, bfs, 0 if gg is g else 1)
                if first is None:
                    first = lv
                assert np.array_equal(lv, first)
            bfs.close()


def test_run_rejects_bad_arguments():
    g = graphgen.from_edges(4, [(0, 1), (1, 2)])
    ro, col = to_dev(g)
    bfs = pkg.S3BFS(ro, col)
    lv = torch.empty(4, dtype=torch.int32, device="cuda")
    pa = torch.empty(4, dtype=torch.int32, device="cuda")
    for s in (-1, 4, 1 << 30):
        with pytest.raises(pkg.S3BFSError) as ei:
            pkg.s3bfs_run(bfs.handle, s, lv, pa)
        assert ei.value.status == 1
    with pytest.raises(ValueError):
        pkg.s3bfs_run(bfs.handle, 0, lv.cpu(), pa)
    bfs.close()


def test_validate_csr_rejects_broken_graphs():
    ro = torch.tensor([0, 2, 1, 3], dtype=torch.int32, device="cuda")   # decreasing
    col = torch.tensor([1, 2, 0], dtype=torch.int32, device="cuda")
    with pytest.raises(pkg.S3BFSError) as ei:
        pkg.S3BFS(ro, col, pkg.Options(validate_csr=1))
    assert ei.value.status == 5
    ro = torch.tensor([0, 1, 2, 3], dtype=torch.int32, device="cuda")
    col = torch.tensor([1, 7, 0], dtype=torch.int32, device="cuda")     # column out of range
    with pytest.raises(pkg.S3BFSError):
        pkg.S3BFS(ro, col, pkg.Options(validate_csr=1))


# ---- (b) the scan alone, bit-exact vs the oracle's exclusive scan --------------------------
SCAN_LENGTHS = [0, 1, 31, 32, 33, 511, 4095, 4096, 4097, 8191, 8193, 65537, 1 << 20,
                (1 << 20) + 1, 1_000_003]


@pytest.mark.parametrize("n", SCAN_LENGTHS)
@pytest.mark.parametrize("dist", ["zeros", "ones", "heavy", "near_max"])
def test_scan_bit_exact(n, dist):
    rng = np.random.default_rng(n * 7 + len(dist))
    if dist == "zeros":
        a = np.zeros(n, np.int32)
    elif dist == "ones":
        a = np.ones(n, np.int32)
    elif dist == "heavy":
        a = np.minimum(rng.pareto(1.2, n) * 3, 60000).astype(np.int32)
    else:  # total just below INT32_MAX
        a = np.full(n, (2**31 - 1) // max(n, 1), np.int32)
    x = torch.from_numpy(a).cuda()
    out = torch.empty(n + 1, dtype=torch.int32, device="cuda")
    pkg.s3bfs_debug_exclusive_scan(x, out)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), oracle.exclusive_scan(a))


def test_scan_2_pow_28():
    n = 1 << 28
    a = np.random.default_rng(5).integers(0, 8, n, dtype=np.int32)
    x = torch.from_numpy(a).cuda()
    out = torch.empty(n + 1, dtype=torch.int32, device="cuda")
    pkg.s3bfs_debug_exclusive_scan(x, out)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), oracle.exclusive_scan(a))


def test_scan_wraps_like_int32():
    a = np.full(10000, 1 << 20, np.int32)   # total 10000 * 2^20 > 2^31: two's-complement wrap
    x = torch.from_numpy(a).cuda()
    out = torch.empty(a.size + 1, dtype=torch.int32, device="cuda")
    pkg.s3bfs_debug_exclusive_scan(x, out)
    want = (np.concatenate([[0], np.cumsum(a.astype(np.int64))]) & 0xFFFFFFFF).astype(np.uint32)
    assert np.array_equal(out.cpu().numpy().view(np.uint32), want)


# ---- (c) the partitioner alone vs the paper's range-marking rule -----------------
@pytest.mark.parametrize("seed", range(6))
def test_find_start_points_vs_range_rule(seed):
    rng = np.random.default_rng(seed)
    n_l = int(rng.integers(1, 200000))
    deg = rng.integers(0, 50, n_l).astype(np.int32)
    deg[rng.random(n_l) < 0.3] = 0          # zero-degree frontier vertices (C9)
    deg[0] = max(deg[0], 1)
    excl = oracle.exclusive_scan(deg)
    e_l = int(excl[-1])
    for p_l in (1, 2, 7, 148, 4096, min(e_l, 100000)):
        chunk = -(-e_l // p_l)
        want_u, want_off = oracle.find_start_points(oracle.inclusive_scan(deg), chunk, p_l)
        ex = torch.from_numpy(excl).cuda()
        u = torch.empty(p_l, dtype=torch.int32, device="cuda")
        off = torch.empty(p_l, dtype=torch.int32, device="cuda")
        pkg.s3bfs_debug_find_start_points(ex, chunk, p_l, u, off)
        torch.cuda.synchronize()
        assert np.array_equal(u.cpu().numpy(), want_u), (seed, p_l)
        assert np.array_equal(off.cpu().numpy(), want_off), (seed, p_l)


def test_find_start_points_spec_examples():
    # SPEC S:238 edge_sum=[2,5,6,10], p_l=2 -> (0,0), (2,0); S:240 [1,2,3,4], p_l=4
    for deg, p_l, wu, wo in (([2, 3, 1, 4], 2, [0, 2], [0, 0]),
                             ([1, 1, 1, 1], 4, [0, 1, 2, 3], [0, 0, 0, 0])):
        excl = oracle.exclusive_scan(np.array(deg, np.int32))
        chunk = -(-int(excl[-1]) // p_l)
        u = torch.empty(p_l, dtype=torch.int32, device="cuda")
        off = torch.empty(p_l, dtype=torch.int32, device="cuda")
        pkg.s3bfs_debug_find_start_points(torch.from_numpy(excl).cuda(), chunk, p_l, u, off)
        assert u.cpu().tolist() == wu and off.cpu().tolist() == wo


# ---- the five BASELINE.json workloads, in the bench's launch configuration ----------------
@pytest.mark.parametrize("cfg,max_sources", [("er", 8), ("grid", 2), ("rmat20", 16),
                                             ("tail", 9), ("rmat24", 3)])
def test_configs_levels_bit_exact(cfg, max_sources):
    g = graphgen.make_config(cfg)
    ro, col = to_dev(g)
    bfs = pkg.S3BFS(ro, col)            # default options = the bench configuration
    for s in g.sources[:max_sources]:
        check_traversal(g, bfs, s)
    bfs.close()
    # NEXT-3: direction-optimising traversal, default switch rule (alpha 14, beta 24)
    bfs = pkg.S3BFS(ro, col, pkg.Options(direction=1))
    for s in g.sources[:max_sources]:
        check_traversal(g, bfs, s)
    bfs.close()


# ---- NEXT-2: clones over one prepared graph, concurrent traversals on separate streams -------
@pytest.mark.parametrize("cfg_kw", [("rmat", dict(debug_poison=1)),
                                    ("rmat", dict(debug_poison=1, direction=1)),
                                    ("grid", dict(debug_poison=1))])
def test_clones_run_concurrently(cfg_kw):
    kind, kw = cfg_kw
    g = graphgen.rmat(14, 16, seed=3) if kind == "rmat" else graphgen.grid(64, 64)
    g.name = kind
    ro, col = to_dev(g)
    base = pkg.S3BFS(ro, col, pkg.Options(**kw))
    clones = [base] + [base.clone() for _ in range(7)]
    srcs = graphgen.pick_sources(g, 8, seed=11)
    streams = [torch.cuda.Stream() for _ in clones]
    outs = []
    for h, st, s in zip(clones, streams, srcs):
        lv = torch.empty(g.n, dtype=torch.int32, device="cuda")
        pa = torch.empty(g.n, dtype=torch.int32, device="cuda")
        pkg.s3bfs_run(h.handle, s, lv, pa, st)
        outs.append((s, lv, pa))
    torch.cuda.synchronize()
    base.close()                      # the prepared graph outlives the source handle
    for (s, lv, pa), h in zip(outs, clones):
        ref, _ = oracle.bfs(g.row_offsets, g.col_indices, s)
        assert np.array_equal(lv.cpu().numpy(), ref)
        assert oracle.check_bfs(g.row_offsets, g.col_indices, s, lv.cpu().numpy(),
                                pa.cpu().numpy())[0] == 0
    for h in clones[1:]:              # clones still usable after the source is gone
        check_traversal(g, h, srcs[0], stats=False)
        h.close()


@pytest.mark.parametrize("kw", [dict(), dict(reorder=-1, tier0_max_edges=-1)],
                         ids=["default", "no-reorder-tier1"])
def test_maximum_size_sparse(kw):
    """Maximum-size edge case: n = 2^28 - 5 (ragged: not a multiple of 32/128/16), a few
    hundred thousand arcs spread over the whole id range (64-bit index arithmetic in create,
    k_init, the relabel sort, the hashed claim slots and k_finalize), a high-id hub and a long
    path crossing the range; levels bit-exact with the oracle, parents by the certificate."""
    n = (1 << 28) - 5
    rng = np.random.default_rng(28)
    hub = n - 1
    path = np.sort(rng.choice(n - 1, 3000, replace=False))
    leaves = rng.choice(n - 1, 100_000, replace=False)
    e = np.concatenate([np.stack([path[:-1], path[1:]], 1),
                        np.stack([np.full(leaves.size, hub), leaves], 1),
                        np.array([[hub, path[0]]])]).astype(np.int64)
    g = graphgen.from_edges(n, e, name="max-sparse")
    ro, col = to_dev(g)
    bfs = pkg.S3BFS(ro, col, pkg.Options(**kw))
    for s in (int(path[-1]), hub, int(leaves[0])):
        check_traversal(g, bfs, s, stats=False)
    unreached = int(np.setdiff1d(np.arange(5), np.concatenate([path, leaves, [hub]]))[0])
    lv, _ = check_traversal(g, bfs, unreached, stats=False)  # isolated source: only itself
    assert (lv >= 0).sum() == 1
    bfs.close()


@pytest.mark.gpu
def test_level_passes_recorded():
    """Level passes (DESIGN R29): a tier-1 level forced into 3 passes is still one stats
    record -- n_l, e_l, kept as the oracle's profile, candidates summed over the passes
    (>= kept), `pad` = the passes it ran (3 where the level has at least 3 edges), and the
    default settings never split a small graph (pad = 1 on every tier-1 level)."""
    g = graphgen.rmat(14, 16, seed=11)
    ro, col = to_dev(g)
    s = graphgen.pick_sources(g, 1, seed=7)[0]
    forced = pkg.S3BFS(ro, col, pkg.Options(debug_poison=1, tag_mode_pct=101, tier0_max_edges=-1,
                                            cluster_max_edges=-1, split_min_edges=1,
                                            split_first_pct=10, split_passes=3))
    check_traversal(g, forced, s)
    st = forced.level_stats()
    t1 = st[st["tier"] == 1]
    assert len(t1) > 0 and np.all(t1["pad"][t1["e_l"] >= 64] == 3), t1["pad"]
    assert np.all((t1["pad"] >= 1) & (t1["pad"] <= 3))
    forced.close()
    plain = pkg.S3BFS(ro, col, pkg.Options(debug_poison=1, tier0_max_edges=-1,
                                           cluster_max_edges=-1))
    check_traversal(g, plain, s)
    st = plain.level_stats()
    assert np.all(st["pad"][st["tier"] == 1] == 1)
    plain.close()


@pytest.mark.parametrize("kw", [dict(collect_stats=-1), dict(collect_stats=-1, loop_mode=2),
                                dict(collect_stats=-1, tier0_max_edges=16)],
                         ids=["graph", "host-loop", "cluster-T0-16"])
def test_stats_off(kw):
    """Per-level statistics off (no level records, tier-0/cluster record counter unused):
    the traversal itself is unchanged."""
    for name, g in TINY + [("rmat12", graphgen.rmat(12, 16, seed=5))]:
        ro, col = to_dev(g)
        bfs = pkg.S3BFS(ro, col, pkg.Options(debug_poison=1, **kw))
        srcs = range(g.n) if g.n <= 16 else sorted({0, g.n // 3, g.n - 1})
        for s in srcs:
            check_traversal(g, bfs, s, stats=False)
        bfs.close()


def test_bounds_checked_build():
    """Memory safety without compute-sanitizer (closed on the GPU pool): the S3BFS_CHECK=1
    build of the same sources checks every data-derived index of the traversal kernels and
    traps on a violation; tests/check_suite.py runs the tiny suite + R-MAT 14/16 under every
    setting of this file through it (and against the oracle) in a fresh process."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    lib = os.path.join(root, "paper_2209_08764_b200", "libs3bfs_check.so")
    assert os.path.exists(lib), "run __graft_entry__.build() (it builds the checked library)"
    env = dict(os.environ, S3BFS_LIB=lib)
    r = subprocess.run([sys.executable, os.path.join(root, "tests", "check_suite.py"), "--quick"],
                       env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "no bounds violation" in r.stdout, (r.stdout[-3000:], r.stderr[-3000:])

"""Experiment: where the first level's fixed cost goes (init -> dispatch -> k_small start)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, graphgen, paper_2209_08764_b200 as pkg
g = graphgen.make_config(sys.argv[1] if len(sys.argv) > 1 else "er")
ro = torch.from_numpy(g.row_offsets).cuda(); col = torch.from_numpy(g.col_indices).cuda()
bfs = pkg.S3BFS(ro, col)
for rep in range(5):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record(); lv, pa = bfs.run(g.sources[0]); ev[1].record(); torch.cuda.synchronize()
    st = bfs.level_stats()
    # read the debug stamps straight from the control block (layout: see s3bfs_kernels.cuh Ctl)
    tl = pkg.s3bfs.s3bfs_debug_timeline(bfs.handle)
    t0 = tl[0]
    print("  init->k_small %.1f us, k_small->L0 end %.1f us" % (
        (tl[2] - t0) / 1e3, (st['t_end_ns'][0] - tl[2]) / 1e3))
    print(f"run {rep}: total {ev[0].elapsed_time(ev[1])*1e3:.1f} us, levels {len(st)}, "
          f"L0 {(st['t_end_ns'][0]-st['t_begin_ns'][0])/1e3:.1f} us, "
          f"L0 end->last level end {(st['t_end_ns'][-1]-st['t_end_ns'][0])/1e3:.1f} us")
# per level: launch gap before k_explore (from the previous level's end), explore, compact
st = bfs.level_stats()
for r in st:
    if r['tier'] == 1:
        print(f"  L{r['level']} tier1 n={r['n_l']} e={r['e_l']}: gap-to-explore "
              f"{(r['t_explore_begin_ns'] - r['t_begin_ns']) / 1e3:.1f} us, explore "
              f"{(r['t_explore_end_ns'] - r['t_explore_begin_ns']) / 1e3:.1f} us, compact+gap "
              f"{(r['t_end_ns'] - r['t_explore_end_ns']) / 1e3:.1f} us")
    else:
        print(f"  L{r['level']} tier{r['tier']} n={r['n_l']} e={r['e_l']}: "
              f"{(r['t_end_ns'] - r['t_begin_ns']) / 1e3:.1f} us")

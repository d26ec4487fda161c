"""Small driver for ncu: one traversal on a BASELINE config (host-loop mode => one launch per
kernel per level, clean per-kernel attribution).  Never a benchmark number."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import graphgen  # noqa: E402
import paper_2209_08764_b200 as pkg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="rmat24")
ap.add_argument("--source-index", type=int, default=0)
ap.add_argument("--loop-mode", type=int, default=2)
ap.add_argument("--runs", type=int, default=1)
ap.add_argument("--all", action="store_true", help="one run from every source of the config")
a = ap.parse_args()
g = graphgen.make_config(a.config)
ro = torch.from_numpy(g.row_offsets).cuda()
col = torch.from_numpy(g.col_indices).cuda()
bfs = pkg.S3BFS(ro, col, pkg.Options(loop_mode=a.loop_mode))
srcs = g.sources if a.all else [g.sources[a.source_index]] * a.runs
for s in srcs:
    level, parent = bfs.run(s)
torch.cuda.synchronize()
st = bfs.level_stats()
for r in st:
    print(f"L{r['level']} n={r['n_l']} e={r['e_l']} tier={r['tier']} grid={r['grid']} "
          f"cand={r['candidates']} us={(r['t_end_ns'] - r['t_begin_ns']) / 1e3:.1f}")
bfs.close()

"""ncu driver (not a benchmark): one direction-optimising R-MAT 24 traversal in host-loop mode
(one launch per kernel per level, so k_bottom_up launches are separable)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import graphgen  # noqa: E402
import paper_2209_08764_b200 as pkg  # noqa: E402

g = graphgen.make_config(sys.argv[1] if len(sys.argv) > 1 else "rmat24")
ro = torch.from_numpy(g.row_offsets).cuda()
col = torch.from_numpy(g.col_indices).cuda()
bfs = pkg.S3BFS(ro, col, pkg.Options(loop_mode=2, direction=1))
bfs.run(g.sources[0])
torch.cuda.synchronize()
for r in bfs.level_stats():
    print(f"L{r['level']} n={r['n_l']} e={r['e_l']} tier={r['tier']} kept={r['kept']} "
          f"us={(r['t_end_ns'] - r['t_begin_ns']) / 1e3:.1f}")

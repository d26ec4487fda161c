"""NEXT-4 on one GPU (experiment record, not a scaling number): G dist ranks stepped in one
process with the loopback exchange, vs the single-GPU handle, on the same sources.  Shows
what the per-level protocol costs (host syncs, record copies, merge kernels) and that every
rank's slice is 1/G of the work.  usage: python scripts/dist_loopback.py CONFIG NSRC G..."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import graphgen  # noqa: E402
import paper_2209_08764_b200 as pkg  # noqa: E402
import paper_2209_08764_b200.dist as pdist  # noqa: E402

cfg, nsrc = sys.argv[1], int(sys.argv[2])
Gs = [int(x) for x in sys.argv[3:]] or [2]
g = graphgen.make_config(cfg)
ro = torch.from_numpy(g.row_offsets).cuda()
col = torch.from_numpy(g.col_indices).cuda()
deg = (ro[1:] - ro[:-1]).to(torch.int64)
srcs = [int(s) for s in g.sources[:nsrc]]
single = pkg.S3BFS(ro, col, pkg.Options(loop_mode=2, tier0_max_edges=-1))
ref = {}
t_single = []
for s in srcs:
    single.run(s)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    lv, _ = single.run(s)
    torch.cuda.synchronize()
    t_single.append(time.perf_counter() - t0)
    ref[s] = lv.cpu().numpy()
print(f"{cfg} single handle (host loop, tier 1 only): {1e3 * np.mean(t_single):.3f} ms/traversal")
for G in Gs:
    ranks = [pdist.DistRank(ro, col, r, G) for r in range(G)]
    tt, ok = [], True
    for s in srcs:
        pdist.traverse(ranks, s)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        outs = pdist.traverse(ranks, s)
        torch.cuda.synchronize()
        tt.append(time.perf_counter() - t0)
        ok &= all(np.array_equal(lv.cpu().numpy(), ref[s]) for lv, _ in outs)
    print(f"{cfg} G={G} loopback (ranks stepped in turn on one GPU): {1e3 * np.mean(tt):.3f} "
          f"ms/traversal, levels equal to the single handle: {ok}")
    for r in ranks:
        r.close()

"""NEXT-2 (multi-source throughput, the paper's many-source protocol P:48): K handles
(1 + K-1 clones over one prepared graph), K streams, traversals round-robin; whole-batch
device time with CUDA events.  Prints one JSON document."""
import argparse
import json
import os
import sys

# K concurrent streams need K hardware work queues (default 8): set before CUDA initialises
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import graphgen  # noqa: E402
import paper_2209_08764_b200 as pkg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="er,grid,rmat20,tail")
ap.add_argument("--ks", default="1,4,16,64")
ap.add_argument("--traversals", type=int, default=128)
ap.add_argument("--direction", type=int, default=0)
ap.add_argument("--stats", type=int, default=-1)
ap.add_argument("--cluster", type=int, default=0, help="options.cluster_max_edges (-1: off)")
a = ap.parse_args()
out = {"what": __doc__.strip().splitlines()[0], "configs": {}}
for cfg in a.configs.split(","):
    g = graphgen.make_config(cfg)
    ro = torch.from_numpy(g.row_offsets).cuda()
    col = torch.from_numpy(g.col_indices).cuda()
    deg = (ro[1:] - ro[:-1]).to(torch.int64)
    base = pkg.S3BFS(ro, col, pkg.Options(direction=a.direction, collect_stats=a.stats,
                                           cluster_max_edges=a.cluster))
    srcs = g.sources
    m_c = {}
    lv = torch.empty(g.n, dtype=torch.int32, device="cuda")
    pa = torch.empty_like(lv)
    for s in srcs:
        base.run(s, lv, pa)
        torch.cuda.synchronize()
        m_c[s] = int(deg[lv >= 0].sum().item())
    res = {}
    for K in [int(k) for k in a.ks.split(",")]:
        hs = [base] + [base.clone() for _ in range(K - 1)]
        sts = [torch.cuda.Stream() for _ in hs]
        bufs = [(torch.empty(g.n, dtype=torch.int32, device="cuda"),
                 torch.empty(g.n, dtype=torch.int32, device="cuda")) for _ in hs]
        for i, (h, st, (l, p)) in enumerate(zip(hs, sts, bufs)):  # warm-up
            pkg.s3bfs_run(h.handle, srcs[i % len(srcs)], l, p, st)
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        for st in sts:
            st.wait_event(ev0)
        edges = 0
        for t in range(a.traversals):
            i = t % K
            s = srcs[t % len(srcs)]
            pkg.s3bfs_run(hs[i].handle, s, bufs[i][0], bufs[i][1], sts[i])
            edges += m_c[s] // 2
        cur = torch.cuda.current_stream()
        for st in sts:
            cur.wait_stream(st)
        ev1.record()
        torch.cuda.synchronize()
        ms = ev0.elapsed_time(ev1)
        res[K] = {"gteps": edges / (ms / 1e3) / 1e9, "ms": ms, "traversals": a.traversals,
                  "traversals_per_s": a.traversals / (ms / 1e3)}
        print(f"{cfg} K={K}: {res[K]['gteps']:.2f} GTEPS, {res[K]['traversals_per_s']:.0f} "
              f"traversals/s", file=sys.stderr, flush=True)
        for h in hs[1:]:
            h.close()
    base.close()
    out["configs"][cfg] = res
print(json.dumps(out))

"""Stress test (experiment): K handles (clones) on K streams running traversals at once,
every result checked against the oracle afterwards.  Used to localise a concurrency fault."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import graphgen  # noqa: E402
import oracle  # noqa: E402
import paper_2209_08764_b200 as pkg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="er")
ap.add_argument("--k", type=int, default=32)
ap.add_argument("--rounds", type=int, default=4)
ap.add_argument("--loop-mode", type=int, default=0)
ap.add_argument("--sync-each", action="store_true")
a = ap.parse_args()
g = graphgen.make_config(a.config)
ro = torch.from_numpy(g.row_offsets).cuda()
col = torch.from_numpy(g.col_indices).cuda()
base = pkg.S3BFS(ro, col, pkg.Options(loop_mode=a.loop_mode))
hs = [base] + [base.clone() for _ in range(a.k - 1)]
sts = [torch.cuda.Stream() for _ in hs]
srcs = g.sources
refs = {s: oracle.bfs(g.row_offsets, g.col_indices, s)[0] for s in srcs}
bad = 0
for r in range(a.rounds):
    outs = []
    for i, (h, st) in enumerate(zip(hs, sts)):
        s = srcs[(i + r) % len(srcs)]
        lv = torch.empty(g.n, dtype=torch.int32, device="cuda")
        pa = torch.empty(g.n, dtype=torch.int32, device="cuda")
        pkg.s3bfs_run(h.handle, s, lv, pa, st)
        if a.sync_each:
            st.synchronize()
        outs.append((s, lv, pa))
    torch.cuda.synchronize()
    for s, lv, pa in outs:
        if not np.array_equal(lv.cpu().numpy(), refs[s]):
            bad += 1
    print(f"round {r}: {len(outs)} traversals, {bad} wrong so far", flush=True)
print("OK" if bad == 0 else f"FAIL {bad}")

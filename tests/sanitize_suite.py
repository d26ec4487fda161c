"""Test infrastructure (may use oracle/; not collected by pytest): the workload the
compute-sanitizer runs (memcheck, synccheck, initcheck, racecheck) execute under
`compute-sanitizer --tool T python tests/sanitize_suite.py [--quick]`.

The tiny suite of tests/test_gpu_parity.py plus R-MAT 14, every tier setting of that file
(single CTA, cluster, tier 1, bottom-up, tag modes, host loop / captured loop), each run
checked against the oracle so a sanitizer run is also a parity run.  The benign race of
PAPER.md:31 (plain Owner / {d, parent} / tag stores by racing discoverers) is a data race by
design at global memory; racecheck covers shared-memory hazards only (tiers 0 and cluster).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import graphgen  # noqa: E402
import oracle  # noqa: E402
import paper_2209_08764_b200 as pkg  # noqa: E402
from test_gpu_parity import SETTINGS, TINY  # noqa: E402

quick = "--quick" in sys.argv
graphs = list(TINY)
g14 = graphgen.rmat(14, 16, seed=9)
g14.name = "rmat14"
graphs.append(("rmat14", g14))
settings = SETTINGS[:6] + SETTINGS[8:12] + SETTINGS[12:14] + SETTINGS[15:17] if quick else SETTINGS
runs = bad = 0
for sname, kw in settings:
    for name, g in graphs:
        ro = torch.from_numpy(g.row_offsets).cuda()
        col = (torch.from_numpy(g.col_indices).cuda() if g.nnz
               else torch.empty(0, dtype=torch.int32, device="cuda"))
        bfs = pkg.S3BFS(ro, col, pkg.Options(**kw))
        srcs = sorted({0, g.n // 2, g.n - 1}) if not quick else [0]
        for s in srcs:
            level, parent = bfs.run(s)
            torch.cuda.synchronize()
            lv, pa = level.cpu().numpy(), parent.cpu().numpy()
            ref, _ = oracle.bfs(g.row_offsets, g.col_indices, s)
            code, _ = oracle.check_bfs(g.row_offsets, g.col_indices, s, lv, pa)
            runs += 1
            if not np.array_equal(lv, ref) or code != 0:
                bad += 1
                print(f"MISMATCH {sname} {name} src {s}", flush=True)
        bfs.close()
print(f"sanitize_suite: {len(settings)} settings x {len(graphs)} graphs, {runs} traversals, "
      f"{bad} mismatches", flush=True)
sys.exit(1 if bad else 0)

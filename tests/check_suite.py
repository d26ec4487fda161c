"""Test infrastructure (may use oracle/): the parity workload of the bounds-checked build.

compute-sanitizer is closed on the GPU pool, so memory safety is checked by a build of the
same sources with S3BFS_CHECK=1 (paper_2209_08764_b200/libs3bfs_check.so, made by
__graft_entry__.build()): every index the traversal kernels derive from data -- frontier
slots, col positions, vertex ids, bitmap words, candidate slots, shared-memory slots -- is
checked against its buffer, and a violation prints the site and traps (the CUDA error then
fails the run).  This driver runs the tiny suite of tests/test_gpu_parity.py plus R-MAT 14
and R-MAT 16 under every tier setting of that file (single CTA, cluster, tier 1, bottom-up,
tag modes, host loop / captured loop), each traversal also checked against the oracle.
usage: S3BFS_LIB=paper_2209_08764_b200/libs3bfs_check.so python tests/check_suite.py [--quick]
(tests/test_gpu_parity.py::test_bounds_checked_build runs it in a subprocess).
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
assert "libs3bfs_check" in pkg.s3bfs.LIB_PATH, "run with S3BFS_LIB=<the bounds-checked build>"
graphs = list(TINY)
for scale in (14, 16):
    g = graphgen.rmat(scale, 16, seed=9)
    g.name = f"rmat{scale}"
    graphs.append((g.name, g))
runs = bad = 0
for sname, kw in SETTINGS:
    for name, g in graphs:
        ro = torch.from_numpy(g.row_offsets).cuda()
        col = (torch.from_numpy(g.col_indices).cuda() if g.nnz
               else torch.empty(0, dtype=torch.int32, device="cuda"))
        bfs = pkg.S3BFS(ro, col, pkg.Options(**kw))
        srcs = [0] if quick else sorted({0, g.n // 2, g.n - 1})
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
print(f"check_suite: {len(SETTINGS)} settings x {len(graphs)} graphs, {runs} traversals, "
      f"{bad} mismatches, no bounds violation", flush=True)
sys.exit(1 if bad else 0)

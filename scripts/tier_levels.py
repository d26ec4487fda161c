"""Experiment record: per-level time by tier and level size (e_l bucket) for option sets.
usage: VARIANT_OPTS='{"name": {...}}' python scripts/tier_levels.py CONFIG NSRC"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import graphgen  # noqa: E402
import paper_2209_08764_b200 as pkg  # noqa: E402

cfg, nsrc = sys.argv[1], int(sys.argv[2])
OPTS = json.loads(os.environ.get("VARIANT_OPTS", '{"default": {}}'))
g = graphgen.make_config(cfg)
ro = torch.from_numpy(g.row_offsets).cuda()
col = torch.from_numpy(g.col_indices).cuda()
buckets = [0, 64, 512, 2048, 4096, 8192, 16384, 32768, 1 << 40]
for name, kw in OPTS.items():
    bfs = pkg.S3BFS(ro, col, pkg.Options(**kw))
    rows = []
    for s in g.sources[:nsrc]:
        bfs.run(int(s))
        torch.cuda.synchronize()
        bfs.run(int(s))
        torch.cuda.synchronize()
        st = bfs.level_stats()
        rows.append(st)
    st = np.concatenate(rows)
    t = (st["t_end_ns"] - st["t_begin_ns"]) / 1e3
    print(f"{cfg} {name}: {len(st)} levels, total {t.sum() / nsrc:.1f} us per source")
    for tier in sorted(set(st["tier"].tolist())):
        for lo, hi in zip(buckets[:-1], buckets[1:]):
            m = (st["tier"] == tier) & (st["e_l"] > lo) & (st["e_l"] <= hi)
            if m.any():
                print(f"   tier {tier} e_l in ({lo},{hi}]: {m.sum():5d} levels, mean {t[m].mean():7.2f} us")
    bfs.close()

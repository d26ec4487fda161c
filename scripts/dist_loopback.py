"""NEXT-4 on one GPU (experiment record, not a scaling number): the 1-D partition's G ranks
stepped in one process (loopback: peers' receive segments and bitmaps are plain device
pointers), each rank's phase timed alone with CUDA events, vs the single-GPU handle (captured
loop) on the same sources.

Per-rank cost model of G GPUs: every level costs max_r explore_r + max_r dedup_r +
max_r advance_r (the ranks' phases run concurrently on their own GPUs) plus the transfer of
the level's remote candidates ({v, parent}, 8 B each) and published bitmap words at the
NVLink 5 rate (900 GB/s per direction per GPU); barriers are not included.  Levels are
checked bit-exact against the single handle.
usage: python scripts/dist_loopback.py CONFIG NSRC G..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import graphgen  # noqa: E402
import paper_2209_08764_b200 as pkg  # noqa: E402
import paper_2209_08764_b200.dist as pdist  # noqa: E402

NVLINK_GBS = 900.0
cfg, nsrc = sys.argv[1], int(sys.argv[2])
Gs = [int(x) for x in sys.argv[3:]] or [2]
g = graphgen.make_config(cfg)
ro = torch.from_numpy(g.row_offsets).cuda()
col = torch.from_numpy(g.col_indices).cuda()
srcs = [int(s) for s in g.sources[:nsrc]]
single = pkg.S3BFS(ro, col)
ref, t_single, cand = {}, [], {}
for s in srcs:
    single.run(s)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    lv, _ = single.run(s)
    b.record()
    torch.cuda.synchronize()
    t_single.append(a.elapsed_time(b))
    ref[s] = lv.cpu().numpy()
    cand[s] = int(single.level_stats()["candidates"].astype(np.int64).sum())
print(f"{cfg} single GPU (captured loop): {np.mean(t_single):.3f} ms/traversal", flush=True)


def timed(fn):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    out = fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b), out


for G in Gs:
    ranks = [pdist.DistRank(ro, col, r, G) for r in range(G)]
    pdist.connect(ranks)
    model, phase, ok = [], {"explore": 0.0, "dedup": 0.0, "advance": 0.0, "xfer": 0.0}, True
    for s in srcs:
        pdist.traverse(ranks, s)  # warm-up
        torch.cuda.synchronize()
        for r in ranks:
            r.begin(s)
        t_model = 0.0
        while True:
            ex = [timed(r.explore)[0] for r in ranks]
            dd = [timed(r.dedup)[0] for r in ranks]
            # (loopback: the phases already ran in rank order, which is the barrier)
            adv = [timed(lambda r=r: r.advance(None, wait=False))[0] for r in ranks]
            t_model += max(ex) + max(dd) + max(adv)
            phase["explore"] += max(ex)
            phase["dedup"] += max(dd)
            phase["advance"] += max(adv)
            if ranks[0].status()[0]:  # the host read, outside the timed phases
                break
        outs = pdist._combine([r.end() for r in ranks], None)
        torch.cuda.synchronize()
        ok &= bool(np.array_equal(outs[0][0].cpu().numpy(), ref[s]))
        # each GPU sends (G-1)/G of its ~1/G share of the candidates (single-GPU count)
        xfer = cand[s] * 8 * (G - 1) / G / G / (NVLINK_GBS * 1e9) * 1e3
        phase["xfer"] += xfer
        model.append(t_model + xfer)
    k = len(srcs)
    print(f"{cfg} G={G}: modelled per-GPU time {np.mean(model):.3f} ms/traversal "
          f"(explore {phase['explore'] / k:.3f}, dedup {phase['dedup'] / k:.3f}, advance "
          f"{phase['advance'] / k:.3f}, NVLink transfer {phase['xfer'] / k:.3f}; max over ranks per "
          f"level, barriers / host syncs excluded) vs single "
          f"{np.mean(t_single):.3f}; levels bit-exact: {ok}", flush=True)
    for r in ranks:
        r.close()

"""Experiment driver (not a benchmark): time design variants of libs3bfs.so on one graph.
usage: python scripts/variants.py CONFIG NSRC tag=path.so [tag=path.so ...]
Each variant x option set: 1 warm-up + 3 timed traversals per source (CUDA events, graph mode);
prints the median per source and the per-level explore/compact split of the last run.
ROUNDS=R repeats the interleaved pass (variants alternate per source) R times."""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import graphgen  # noqa: E402
from paper_2209_08764_b200.s3bfs import LevelStat, Options  # noqa: E402

cfg, nsrc = sys.argv[1], int(sys.argv[2])
variants = [a.split("=", 1) for a in sys.argv[3:]]
OPTS = json.loads(os.environ.get("VARIANT_OPTS", '{"default": {}, "nohot": {"hot_min_edges": -1}}'))
g = graphgen.make_config(cfg)
ro = torch.from_numpy(g.row_offsets).cuda()
col = torch.from_numpy(g.col_indices).cuda()
deg = (ro[1:] - ro[:-1]).to(torch.int64)
level = torch.empty(g.n, dtype=torch.int32, device="cuda")
parent = torch.empty(g.n, dtype=torch.int32, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream()
vp = ctypes.c_void_p
results = {}
ROUNDS = int(os.environ.get("ROUNDS", "1"))
handles = []  # (key, lib, handle): every variant is created up front, then runs interleave
for tag, path in variants:
    lib = ctypes.CDLL(os.path.abspath(path))
    lib.s3bfs_create.argtypes = [ctypes.POINTER(vp), ctypes.c_int32, ctypes.c_int64, vp, vp,
                                 ctypes.POINTER(Options), vp]
    lib.s3bfs_run.argtypes = [vp, ctypes.c_int32, vp, vp, vp]
    lib.s3bfs_destroy.argtypes = [vp]
    lib.s3bfs_get_level_stats.argtypes = [vp, ctypes.POINTER(LevelStat), ctypes.c_int32,
                                          ctypes.POINTER(ctypes.c_int32)]
    for oname, okw in OPTS.items():
        h = vp()
        o = Options(**okw)
        rc = lib.s3bfs_create(ctypes.byref(h), g.n, g.nnz, ro.data_ptr(), col.data_ptr(),
                              ctypes.byref(o), st.cuda_stream)
        assert rc == 0, rc
        handles.append((f"{tag}/{oname}", lib, h))
srcs = list(g.sources[:nsrc])
times = {k: {s: [] for s in srcs} for k, _, _ in handles}
levels = {k: {} for k, _, _ in handles}
edges = {}
for rnd in range(ROUNDS):
    for s in srcs:
        for key, lib, h in handles:  # interleaved: clock drift hits every variant alike
            for rep in range(4 if rnd == 0 else 3):
                flush.fill_(rep)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(st)
                assert lib.s3bfs_run(h, s, level.data_ptr(), parent.data_ptr(), st.cuda_stream) == 0
                b.record(st)
                b.synchronize()
                if rep or rnd:
                    times[key][s].append(a.elapsed_time(b))
            if s not in edges:
                edges[s] = int(deg[level >= 0].sum().item()) // 2
            buf = (LevelStat * 256)()
            num = ctypes.c_int32()
            lib.s3bfs_get_level_stats(h, buf, 256, ctypes.byref(num))
            levels[key][s] = [(r.level, r.e_l, r.tier, (r.t_explore_end_ns - r.t_explore_begin_ns) / 1e3,
                               (r.t_end_ns - r.t_explore_end_ns) / 1e3 if r.tier == 1 else 0.0,
                               r.candidates, r.kept) for r in buf[: min(num.value, 256)]]
for key, lib, h in handles:
    lib.s3bfs_destroy(h)
    per = [{"src": s, "ms": float(np.median(times[key][s])), "gteps": edges[s] / float(np.median(times[key][s])) / 1e6,
            "heavy": [x for x in levels[key][s] if x[1] > 1_000_000]} for s in srcs]
    tot_ms = sum(p["ms"] for p in per)
    tot_e = sum(edges[s] for s in srcs)
    results[key] = {"gteps": tot_e / tot_ms / 1e6, "per": per}
    t1 = [x for s in srcs for x in levels[key][s] if x[2] == 1]
    kx_us = sum(x[3] for x in t1)
    kc_us = sum(x[4] for x in t1)
    alg = sum(8 * x[1] + 16 * x[5] for x in t1)
    frac = alg / (kx_us * 1e-6) / 6.5498e12 if kx_us else 0.0
    print(f"{key:32s} GTEPS {tot_e / tot_ms / 1e6:7.2f}  kx {kx_us:8.0f} us kc {kc_us:7.0f} us "
          f"frac(kx, in-graph) {frac:.3f}  ms/src " + " ".join(f"{p['ms']:.3f}" for p in per),
          flush=True)
    worst = max(per, key=lambda p: p["ms"])
    for p in per[:2] + ([worst] if worst not in per[:2] else []):
        print("    src", p["src"], " ".join(f"[e={x[1]/1e6:.1f}M kx={x[3]:.0f} kc={x[4]:.0f} c={x[5]/1e6:.2f}M k={x[6]/1e6:.2f}M]"
                                           for x in p["heavy"]), flush=True)
json.dump(results, open(os.environ.get("VARIANT_OUT", "gpurun_out/variants.json"), "w"))

"""NEXT-1: the paper's experiment (Fig. 2a) replayed on one B200.

Work-sensitive S3BFS (variant 0: P_l = min(P_max, ceil(e_l/grain)), single-CTA tier for tiny
levels) vs work-insensitive (variant 1: every level on the full grid P_max), same graph and
sources.  Reports the per-level time ratio insensitive/sensitive (> 1 = work-sensitive
faster; the paper reports per-level performance ratios the same way round) from the
library's %globaltimer level stamps, whole-traversal times from CUDA events, and the energy
per traversal from NVML's total-energy counter over a long loop of repeated traversals.
Output: one JSON document (stdout)."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import graphgen  # noqa: E402
import paper_2209_08764_b200 as pkg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="er,rmat20,rmat24")
ap.add_argument("--sources", type=int, default=4)
ap.add_argument("--energy-seconds", type=float, default=3.0)
a = ap.parse_args()

try:
    import pynvml
    pynvml.nvmlInit()
    nvh = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
except Exception:  # noqa: BLE001
    nvh = None


def energy_mj():
    return pynvml.nvmlDeviceGetTotalEnergyConsumption(nvh) if nvh is not None else None


out = {"what": __doc__.strip().splitlines()[0], "configs": {}}
for cfg in a.configs.split(","):
    g = graphgen.make_config(cfg)
    ro = torch.from_numpy(g.row_offsets).cuda()
    col = torch.from_numpy(g.col_indices).cuda()
    res = {}
    for name, variant in (("work_sensitive", 0), ("work_insensitive", 1)):
        bfs = pkg.S3BFS(ro, col, pkg.Options(variant=variant))
        lvl = torch.empty(g.n, dtype=torch.int32, device="cuda")
        par = torch.empty_like(lvl)
        per_src = []
        for s in g.sources[: a.sources]:
            for _ in range(2):
                bfs.run(s, lvl, par)
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            ev[0].record()
            reps = 5
            for _ in range(reps):
                bfs.run(s, lvl, par)
            ev[1].record()
            torch.cuda.synchronize()
            st = bfs.level_stats()
            per_src.append({"source": int(s), "ms": ev[0].elapsed_time(ev[1]) / reps,
                            "level_us": ((st["t_end_ns"] - st["t_begin_ns"]) / 1e3).tolist(),
                            "n_l": st["n_l"].tolist(), "e_l": st["e_l"].tolist(),
                            "tier": st["tier"].tolist(), "grid": st["grid"].tolist()})
        # energy: repeat traversals over the sources for ~energy_seconds
        torch.cuda.synchronize()
        e0, t0, runs = energy_mj(), time.perf_counter(), 0
        while time.perf_counter() - t0 < a.energy_seconds:
            for s in g.sources[: a.sources]:
                bfs.run(s, lvl, par)
                runs += 1
            torch.cuda.synchronize()
        e1, t1 = energy_mj(), time.perf_counter()
        bfs.close()
        res[name] = {"per_source": per_src, "runs_for_energy": runs,
                     "mj_per_traversal": (e1 - e0) / runs if e0 is not None else None,
                     "avg_power_w": (e1 - e0) / 1e3 / (t1 - t0) if e0 is not None else None}
    ratios = []
    for ps, pi in zip(res["work_sensitive"]["per_source"], res["work_insensitive"]["per_source"]):
        r = [i / s if s > 0 else None for s, i in zip(ps["level_us"], pi["level_us"])]
        ratios.append({"source": ps["source"], "traversal_ratio": pi["ms"] / ps["ms"],
                       "per_level_ratio": r, "n_l": ps["n_l"], "e_l": ps["e_l"]})
    ws, wi = res["work_sensitive"], res["work_insensitive"]
    out["configs"][cfg] = {
        "ratios_insensitive_over_sensitive": ratios,
        "energy_ratio_insensitive_over_sensitive":
            (wi["mj_per_traversal"] / ws["mj_per_traversal"]) if ws["mj_per_traversal"] else None,
        "detail": res}
    print(f"{cfg}: traversal time ratio (insens/sens) " +
          " ".join(f"{r['traversal_ratio']:.2f}" for r in ratios) +
          f"; energy ratio {out['configs'][cfg]['energy_ratio_insensitive_over_sensitive']}",
          file=sys.stderr, flush=True)
print(json.dumps(out))

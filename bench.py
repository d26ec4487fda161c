#!/usr/bin/env python
"""Benchmark: BFS GTEPS per source on one B200 (+ expansion-kernel roofline), BASELINE.json.

A "step" is one full traversal s3bfs_run(source) -- every row of SURVEY.md s.8(a) -- on the
workload BASELINE.json's metric is quoted on: R-MAT scale 24, edge factor 16 (configs[3]),
cycling over its 16 seeded non-isolated sources.  The graph (2.08 GB of col_indices) is
resident in HBM before timing; the L2 is also flushed (256 MB write) before every step,
outside that step's CUDA-event pair.

Legs (all printed in ONE JSON line by rank 0):
  value        device-timed GTEPS = sum over steps and ranks of m_c/2 / max-over-ranks time
  e2e          the same through the C ABI with the result read back to pinned host memory
  roofline     k_explore (the dominant kernel): algorithmic bytes / CUDA-event duration, from
               a host-loop pass with per-launch events
  cpu_baseline the oracle (serial C BFS) on a bounded sample of the same sources, 1 core
--impl reference times the oracle alone as the reference arm (rank 0 only).
Multi-GPU (torchrun): independent traversals per rank (replicas, weak scaling); the only
collectives are the timing barrier and the max-over-ranks reduction.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "BFS GTEPS per source on 1 B200; expansion-kernel HBM GB/s as % of peak"
CONFIG_INDEX = {"er": 0, "grid": 1, "rmat20": 2, "rmat24": 3, "tail": 4}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=128)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="s3bfs", choices=["s3bfs", "reference"])
    ap.add_argument("--config", default="rmat24", choices=list(CONFIG_INDEX))
    ap.add_argument("--oracle-sources", type=int, default=3,
                    help="sources checked bit-exactly against (and timed on) the oracle")
    ap.add_argument("--no-flush", action="store_true")
    ap.add_argument("--detail-out", default="")
    ap.add_argument("--loop-mode", type=int, default=0)
    ap.add_argument("--tier0", type=int, default=0)
    ap.add_argument("--grain", type=int, default=0)
    ap.add_argument("--next4", action="store_true",
                    help="multi-GPU nodes: also time ONE traversal split over all ranks (NEXT-4, "
                         "1-D vertex partition, peer-memory exchange; strong scaling), reported "
                         "beside the line")
    ap.add_argument("--no-next3", action="store_true",
                    help="skip the extra direction-optimising (NEXT-3) measurement")
    ap.add_argument("--direction", type=int, default=0,
                    help="1: direction-optimising traversal (NEXT-3); default: the paper's top-down")
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.samples = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "10"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            time.sleep(0.3)
        except Exception:  # noqa: BLE001
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.samples.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:  # noqa: BLE001
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def launches_from_stats(st, td_chain: int = 1, bu_chain: int = 1, universal: int = 0,
                        direction: int = 0, prologue: int = 0) -> int:
    """Kernel launches of one traversal in graph mode, replaying the captured loop over the
    level tiers: k_init; per WHILE iteration the SWITCH body of the current level's tier --
    S (k_small: a whole run of tier-0 levels), C (k_cluster: a whole run of cluster levels),
    T (k_explore + k_compact: one top-down level), B (k_fb_clear + k_fb_set + k_bottom_up:
    one bottom-up level, NEXT-3) -- where a body is its own tier (T x td_chain, B x bu_chain)
    or, universal, the sequence S C T^td [B^bu T^td] C S from its tier on; with prologue that
    whole sequence first runs once between k_init and the loop; every kernel of a chain
    launches (idle ones return at once); then k_finalize."""
    # a tier-1 level that ran as p passes (level passes, `pad` of its record) is p T entries
    try:
        passes = [int(p) for p in st["pad"]]
    except (KeyError, ValueError, IndexError):
        passes = [1] * len(st["tier"])
    tiers = []
    for t, p in zip(st["tier"], passes):
        if t in (0, 1, 3, 4):
            tiers += [{0: "S", 1: "T", 3: "B", 4: "C"}[int(t)]] * (max(1, p) if int(t) == 1 else 1)
    seq = "SC" + "T" * td_chain + ("B" * bu_chain + "T" * td_chain if direction else "") + "CS"
    cost = {"S": 1, "C": 1, "T": 2, "B": 3}
    n, i, first = 1, 0, bool(prologue)
    while i < len(tiers) or first:
        t = tiers[i] if i < len(tiers) else "S"
        body = (seq if first else seq[seq.index(t):] if universal
                else t * (td_chain if t == "T" else bu_chain if t == "B" else 1))
        first = False
        for k in body:
            n += cost[k]
            if i < len(tiers) and tiers[i] == k:
                i += 1
                while k in "SC" and i < len(tiers) and tiers[i] == k:
                    i += 1
    return n + 1


def shard_sources(srcs, rank: int, world: int) -> list:
    """Rank r's traversal order: the config's sources rotated by r (replicas, weak scaling:
    every rank runs the same number of independent traversals, no data-path collective)."""
    return [srcs[(rank + k) % len(srcs)] for k in range(len(srcs))]


def job_throughput(my_ms: float, my_edges: float, dev, world: int):
    """Whole-job GTEPS: edges summed over ranks / device time max-reduced over ranks.
    Returns (gteps, max_ms, total_edges).  Plain values when world == 1."""
    import torch
    t = torch.tensor([my_ms], dtype=torch.float64, device=dev)
    e = torch.tensor([my_edges], dtype=torch.float64, device=dev)
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(e, op=dist.ReduceOp.SUM)
    max_ms, tot = float(t.item()), float(e.item())
    return tot / (max_ms / 1e3) / 1e9, max_ms, tot


def cpu_baseline(g, srcs, args, flags, per):
    """the oracle (serial FIFO BFS) on the host cores, same CSR in host memory,
    same sources.  Single core: per source the median of 3 runs; value = sum of m_c/2 over
    the sample / sum of the medians.  Throughput: N threads at once, each its own source (no
    shared mutable state), aggregate m_c/2 over the wall time; N = min(cores, sources)."""
    import concurrent.futures as cf

    import oracle
    sample = srcs[: max(1, min(args.oracle_sources, len(srcs)))]
    meds, edges = [], 0
    for s in sample:
        reps = []
        for _ in range(3):
            t0 = time.perf_counter()
            oracle.bfs(g.row_offsets, g.col_indices, s)
            reps.append(time.perf_counter() - t0)
        meds.append(statistics.median(reps))
        edges += per[s]["m_c"] // 2
    single = edges / sum(meds) / 1e9
    cores = os.cpu_count() or 1
    nthr = max(1, min(cores, len(srcs)))
    tp_srcs = [srcs[k % len(srcs)] for k in range(nthr)]
    t0 = time.perf_counter()
    with cf.ThreadPoolExecutor(nthr) as ex:  # ctypes drops the GIL inside oracle_bfs
        list(ex.map(lambda s: oracle.bfs(g.row_offsets, g.col_indices, s), tp_srcs))
    wall = time.perf_counter() - t0
    tp = sum(per[s]["m_c"] // 2 for s in tp_srcs) / wall / 1e9
    return {"value": single, "unit": "GTEPS", "cores": 1, "kind": "oracle",
            "sample": f"oracle_bfs (serial FIFO BFS, {flags}), median of 3 runs from each of "
                      f"the first {len(sample)} of {len(srcs)} {args.config} sources "
                      f"({3 * sum(meds):.1f} s of CPU work)",
            "cpu_model": oracle.cpu_model(), "host_cores_total": cores,
            "throughput": {"value": tp, "unit": "GTEPS", "threads": nthr,
                           "what": f"{nthr} host threads at once, each one traversal from its "
                                   f"own source (the config's sources in order); aggregate "
                                   f"m_c/2 over the wall time ({wall:.1f} s)"},
            "median_ms_per_source": [m * 1e3 for m in meds]}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import graphgen
    import oracle
    g = graphgen.make_config(args.config)
    srcs = g.sources
    budget_s = 150.0
    warm = min(args.warmup, 1)
    for i in range(warm):
        oracle.bfs(g.row_offsets, g.col_indices, srcs[i % len(srcs)])
    done, edges, t_tot = 0, 0, 0.0
    for k in range(args.steps):
        s = srcs[k % len(srcs)]
        t0 = time.perf_counter()
        lv, _ = oracle.bfs(g.row_offsets, g.col_indices, s)
        dt = time.perf_counter() - t0
        _, _, m_c, _ = oracle.level_profile(g.row_offsets, lv)
        done += 1
        edges += m_c // 2
        t_tot += dt
        if t_tot > budget_s:
            break
    gteps = edges / t_tot / 1e9
    sample = (f"oracle_bfs (serial FIFO BFS, C -O3, 1 thread) on {args.config}: {done} of "
              f"{args.steps} steps (150 s budget), warmup {warm}")
    line = {"impl": "reference", "metric": METRIC, "value": gteps, "unit": "GTEPS",
            "n_gpus": args.gpus, "steps": done, "warmup": warm,
            "ms_per_step": t_tot / done * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "int32", "data": "synthetic (seeded graphgen)",
            "config": {"workload": args.config, "baseline_config": CONFIG_INDEX[args.config],
                       "n": g.n, "nnz": g.nnz},
            "cpu_baseline": {"value": gteps, "unit": "GTEPS", "cores": 1, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": gteps, "unit": "GTEPS", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    import graphgen
    import paper_2209_08764_b200 as pkg

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    threads = max(1, (os.cpu_count() or 8) // max(world, 1))
    g = graphgen.make_config(args.config, threads=threads)
    ro = torch.from_numpy(g.row_offsets).to(dev)
    col = torch.from_numpy(g.col_indices).to(dev)
    deg = (ro[1:] - ro[:-1]).to(torch.int64)
    opts = pkg.Options(loop_mode=args.loop_mode, tier0_max_edges=args.tier0,
                       edges_per_cta=args.grain, direction=args.direction)
    bfs = pkg.S3BFS(ro, col, opts)
    info = bfs.info()
    n = g.n
    level = torch.empty(n, dtype=torch.int32, device=dev)
    parent = torch.empty(n, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream(dev)
    sp = int(stream.cuda_stream)
    lp, pp = int(level.data_ptr()), int(parent.data_ptr())

    # ---- untimed: per-source edge counts (m_c from the traversal's own levels), launches,
    # and bit-exact oracle checks + CPU baseline on a bounded sample of sources ------------
    srcs = g.sources
    my_srcs = shard_sources(srcs, rank, world)
    per = {}
    for s in sorted(set(my_srcs)):
        pkg.s3bfs_run_ptr(bfs.handle, s, lp, pp, sp)
        st = bfs.level_stats()
        m_c = int(deg[level >= 0].sum().item())
        per[s] = {"m_c": m_c, "levels": int(len(st)), "launches": launches_from_stats(
            st, *((info["td_chain"], info["bu_chain"], info["universal_body"], args.direction,
                   info["prologue"]) if args.loop_mode != 2 else (1, 1, 0, 0, 0))),
                  "stats": st}
    verified = {"sources": 0, "levels_bit_exact": True, "parents_valid": True}
    cpu = None
    oracle_levels = {}
    if rank == 0 and args.oracle_sources > 0:
        import oracle
        flags = oracle.use_native()  # -O3 -march=native, built on this host
        for s in srcs[: args.oracle_sources]:
            pkg.s3bfs_run_ptr(bfs.handle, s, lp, pp, sp)
            torch.cuda.synchronize()
            lv, pa = level.cpu().numpy(), parent.cpu().numpy()
            ref, _ = oracle.bfs(g.row_offsets, g.col_indices, s)
            oracle_levels[s] = ref
            ok = bool(np.array_equal(lv, ref))
            code, _ = oracle.check_bfs(g.row_offsets, g.col_indices, s, lv, pa)
            _, _, m_c, _ = oracle.level_profile(g.row_offsets, ref)
            verified["sources"] += 1
            verified["levels_bit_exact"] &= ok and m_c == per[s]["m_c"]
            verified["parents_valid"] &= code == 0
        if not (verified["levels_bit_exact"] and verified["parents_valid"]):
            print(f"VERIFICATION FAILED: {verified}", file=sys.stderr, flush=True)
        cpu = cpu_baseline(g, srcs, args, flags, per)

    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def one_step(k, ev0=None, ev1=None):
        s = my_srcs[k % len(my_srcs)]
        if not args.no_flush:
            flush_buf.fill_(k & 255)
        if ev0 is not None:
            ev0.record(stream)
        pkg.s3bfs_run_ptr(bfs.handle, s, lp, pp, sp)
        if ev1 is not None:
            ev1.record(stream)
        return s

    for k in range(args.warmup):
        one_step(k)
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        done_srcs = [one_step(k, *evs[k]) for k in range(args.steps)]
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    my_ms = float(sum(step_ms))
    my_edges = sum(per[s]["m_c"] // 2 for s in done_srcs)
    my_launches = sum(per[s]["launches"] for s in done_srcs)
    value, max_ms, tot_edges = job_throughput(my_ms, my_edges, dev, world)
    per_step_gteps = [per[s]["m_c"] / 2 / (ms / 1e3) / 1e9 for s, ms in zip(done_srcs, step_ms)]
    hmean = len(per_step_gteps) / sum(1.0 / x for x in per_step_gteps)

    # ---- e2e: through the C ABI, every step's result read back to pinned host memory -------
    # (a) serial: each step's traversal + its D2H copy timed alone (reported in detail);
    # (b) the e2e value: the same steps as one stream of work, each step's copy (copy stream)
    #     overlapping the next step's traversal on double-buffered outputs -- every step's
    #     transfer is inside the one timed region.  col (2 GB) exceeds L2: no flush needed.
    h_lv = [torch.empty(n, dtype=torch.int32, pin_memory=True) for _ in range(2)]
    h_pa = [torch.empty(n, dtype=torch.int32, pin_memory=True) for _ in range(2)]
    e2e_steps = min(args.steps, 16)
    ser_ms, e2e_edges = 0.0, 0
    for k in range(e2e_steps):
        if not args.no_flush:
            flush_buf.fill_(k & 255)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        s = my_srcs[k % len(my_srcs)]
        pkg.s3bfs_run_ptr(bfs.handle, s, lp, pp, sp)
        h_lv[0].copy_(level, non_blocking=True)
        h_pa[0].copy_(parent, non_blocking=True)
        b.record(stream)
        b.synchronize()
        ser_ms += a.elapsed_time(b)
        e2e_edges += per[s]["m_c"] // 2
    ser_value, _, _ = job_throughput(ser_ms, e2e_edges, dev, world)
    d_lv = [level, torch.empty_like(level)]
    d_pa = [parent, torch.empty_like(parent)]
    cstream = torch.cuda.Stream(dev)
    copied = [torch.cuda.Event(), torch.cuda.Event()]
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for k in range(e2e_steps):
        i = k & 1
        if k >= 2:
            stream.wait_event(copied[i])  # buffer i's previous result is on the host
        s = my_srcs[k % len(my_srcs)]
        pkg.s3bfs_run_ptr(bfs.handle, s, int(d_lv[i].data_ptr()), int(d_pa[i].data_ptr()), sp)
        done = torch.cuda.Event()
        done.record(stream)
        cstream.wait_event(done)
        with torch.cuda.stream(cstream):
            h_lv[i].copy_(d_lv[i], non_blocking=True)
            h_pa[i].copy_(d_pa[i], non_blocking=True)
        copied[i].record(cstream)
    stream.wait_stream(cstream)
    b.record(stream)
    b.synchronize()
    e2e_ms = a.elapsed_time(b)
    e2e_value, _, _ = job_throughput(e2e_ms, e2e_edges, dev, world)
    e2e_ok = all(bool(torch.equal(h_lv[(e2e_steps - 1 - j) & 1],
                                  d_lv[(e2e_steps - 1 - j) & 1].cpu())) for j in range(2))

    # ---- NEXT-3: the same steps with the direction-optimising option (not the headline) ----
    next3 = None
    if not args.direction and not args.no_next3:
        hd = pkg.S3BFS(ro, col, pkg.Options(direction=1, loop_mode=args.loop_mode))
        d_ok = True
        for s, ref in oracle_levels.items():  # bit-exact against the oracle too
            pkg.s3bfs_run_ptr(hd.handle, s, lp, pp, sp)
            torch.cuda.synchronize()
            d_ok &= bool(np.array_equal(level.cpu().numpy(), ref))
        for k in range(args.warmup):
            pkg.s3bfs_run_ptr(hd.handle, my_srcs[k % len(my_srcs)], lp, pp, sp)
        torch.cuda.synchronize()
        d_ms, d_edges = 0.0, 0
        for k in range(args.steps):
            s = my_srcs[k % len(my_srcs)]
            if not args.no_flush:
                flush_buf.fill_(k & 255)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            pkg.s3bfs_run_ptr(hd.handle, s, lp, pp, sp)
            b.record(stream)
            b.synchronize()
            d_ms += a.elapsed_time(b)
            d_edges += per[s]["m_c"] // 2
        d_value, d_max_ms, _ = job_throughput(d_ms, d_edges, dev, world)
        hd.close()
        next3 = {"what": "direction-optimising traversal (SURVEY NEXT-3, option direction=1; "
                         "Beamer switch alpha=14 beta=24), same sources/steps/flushes",
                 "value": d_value, "unit": "GTEPS", "ms_per_step": d_max_ms / args.steps,
                 "levels_bit_exact_vs_oracle": d_ok, "sources_checked": len(oracle_levels)}

    # ---- NEXT-4 (opt-in, world > 1): one traversal split over all ranks, strong scaling ----
    next4 = None
    if args.next4 and world > 1:
        import paper_2209_08764_b200.dist as pdist
        dr = pdist.DistRank(ro, col, rank, world)
        pdist.connect([dr], dist.group.WORLD)  # exchange records; peers opened by CUDA IPC
        n4_steps = min(args.steps, 16)
        checked = [s for s in srcs[: args.oracle_sources] if s in oracle_levels]
        n4_ok = True if checked else None
        for s in srcs[: args.oracle_sources]:  # every rank traverses (collectives); rank 0 checks
            (lv4, _), = pdist.traverse([dr], s, group=dist.group.WORLD)
            torch.cuda.synchronize()
            if s in oracle_levels:
                n4_ok &= bool(np.array_equal(lv4.cpu().numpy(), oracle_levels[s]))
        # m_c / 2 per source from the single-GPU traversals (outside the timed region)
        mc_half = {s: p["m_c"] // 2 for s, p in per.items()}
        for k in range(args.warmup):
            pdist.traverse([dr], srcs[k % len(srcs)], group=dist.group.WORLD)
        torch.cuda.synchronize()
        dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        n4_edges = 0
        for k in range(n4_steps):  # every rank runs the SAME source (one traversal)
            pdist.traverse([dr], srcs[k % len(srcs)], group=dist.group.WORLD)
            n4_edges += mc_half[srcs[k % len(srcs)]]
        b.record(stream)
        torch.cuda.synchronize()
        t = torch.tensor([a.elapsed_time(b)], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dr.close()
        next4 = {"what": "SURVEY NEXT-4: one traversal over all ranks, 1-D vertex partition "
                         "(candidates stored into the owners' receive segments by the "
                         "exploration kernel over NVLink peer memory, owner-side Owner check, "
                         "replicated bitmap words published by peer stores; NCCL one-element "
                         "all-reduces order the phases); same sources, no L2 flush",
                 "value": n4_edges / (float(t.item()) / 1e3) / 1e9, "unit": "GTEPS",
                 "ranks": world, "scaling": "strong",
                 "ms_per_traversal": float(t.item()) / n4_steps,
                 "levels_bit_exact_vs_oracle": n4_ok}

    # ---- roofline of k_explore: per-launch CUDA events (host-loop pass, same kernels) -----
    roof = None
    detail = {}
    if rank == 0:
        hb = pkg.S3BFS(ro, col, pkg.Options(loop_mode=2, time_kernels=1,
                                            tier0_max_edges=args.tier0,
                                            edges_per_cta=args.grain, direction=args.direction))
        ex_ms, ex_launch, alg_bytes, cm_ms, sm_ms = 0.0, 0, 0, 0.0, 0.0
        step_ms_hl = 0.0
        for s in srcs:
            flush_buf.fill_(1)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            hb.run(s, level, parent)
            kt = pkg.s3bfs_get_kernel_times(hb.handle)
            step_ms_hl += (time.perf_counter() - t0) * 1e3
            st = hb.level_stats()
            t1 = st[st["tier"] == 1]
            # SURVEY s.8(d): Kd = 4 B/arc col stream + 4 B/arc status + 16 B per discovery
            alg_bytes += int(8 * t1["e_l"].astype(np.int64).sum()
                             + 16 * t1["candidates"].astype(np.int64).sum())
            ex_ms += kt["explore_ms"]
            ex_launch += kt["explore_launches"]
            cm_ms += kt["compact_ms"]
            sm_ms += kt["small_ms"]
        hb.close()
        peak, peak_src = peaks()
        achieved = alg_bytes / ex_launch / (ex_ms / ex_launch / 1e3) / 1e9 if ex_ms else 0.0
        # the same kernel inside the captured loop (globaltimer, CTA-0 start stamps)
        in_graph_ms = sum(float(((p["stats"]["t_explore_end_ns"] - p["stats"]["t_explore_begin_ns"])
                                 [p["stats"]["tier"] == 1]).sum()) / 1e6 for p in per.values())
        step_total = sum(float(p["stats"]["t_end_ns"][-1] - p["stats"]["t_begin_ns"][0]) / 1e6
                         for p in per.values())
        # ncu-measured DRAM bytes per k_explore launch (profiles/ncu_traffic.json, keyed by
        # config; written by scripts/ncu_traffic.py from an ncu capture of this bench command)
        traffic, traffic_detail = None, None
        tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(tp):
            try:
                traffic_detail = json.load(open(tp)).get(args.config)
                traffic = traffic_detail["dram_bytes_per_launch"] if traffic_detail else None
            except Exception:  # noqa: BLE001
                traffic, traffic_detail = None, None
        # per tier-1 level (in-graph CTA-0 stamps of the bench's own traversals): the same
        # algorithmic bytes over that level's k_explore span, for the levels that carry the work
        lvl = []
        for s_, p in per.items():
            stt = p["stats"]
            for r in stt[(stt["tier"] == 1) & (stt["e_l"] >= 1_000_000)]:
                us = float(r["t_explore_end_ns"] - r["t_explore_begin_ns"]) / 1e3
                b = 8 * int(r["e_l"]) + 16 * int(r["candidates"])
                lvl.append({"source": int(s_), "level": int(r["level"]), "e_l": int(r["e_l"]),
                            "candidates": int(r["candidates"]), "us": us,
                            "frac": b / (us * 1e-6) / (peak * 1e9) if us > 0 else None})
        detail["heavy_levels"] = lvl
        fr = sorted(x["frac"] for x in lvl if x["frac"])
        roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic, "kernel": "k_explore",
                "frac_of_8tbs": achieved / 8000.0,
                "traffic_detail": traffic_detail,
                "heavy_level_frac": ({"levels": len(fr), "min": fr[0], "median": fr[len(fr) // 2],
                                      "max": fr[-1], "what": "tier-1 levels with e_l >= 1e6, "
                                      "in-graph CTA-0 stamps, same byte model"} if fr else None),
                "peak_source": peak_src, "launches": ex_launch,
                "bytes_per_launch": alg_bytes / max(ex_launch, 1),
                "avg_launch_ms": ex_ms / max(ex_launch, 1),
                "share_of_step_events": ex_ms / max(ex_ms + cm_ms + sm_ms, 1e-9),
                "share_of_step_in_graph": in_graph_ms / max(step_total, 1e-9),
                "compact_ms_total": cm_ms, "small_ms_total": sm_ms}
        detail["roofline_pass"] = {"explore_ms": ex_ms, "compact_ms": cm_ms, "small_ms": sm_ms,
                                   "host_loop_wall_ms": step_ms_hl}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GTEPS", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": max_ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "int32", "data": f"synthetic (seeded graphgen {args.config}, BASELINE.json "
                                      f"configs[{CONFIG_INDEX[args.config]}])",
            "config": {"workload": args.config, "baseline_config": CONFIG_INDEX[args.config],
                       "n": g.n, "nnz": g.nnz, "sources": len(srcs),
                       "l2": "flushed (256 MB write) before every step, outside its events"
                             if not args.no_flush else "not flushed (col 2 GB > L2)",
                       "loop": "cuda-graph" if args.loop_mode != 2 else "host",
                       "p_max": info["p_max"], "grain": info["edges_per_cta"],
                       "t0": info["tier0_max_edges"],
                       "direction": "optimising (NEXT-3)" if args.direction else "top-down (S3BFS)"},
            "gteps_hmean": hmean, "gteps_min": min(per_step_gteps),
            "gteps_max": max(per_step_gteps),
            "roofline": roof, "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "GTEPS", "h2d_bytes_per_step": 4,
                    "d2h_bytes_per_step": 8 * n, "steps": e2e_steps,
                    "what": "s3bfs_run through the C ABI (source by value) + level/parent "
                            "copied to pinned host memory every step; the steps as one "
                            "timed stream, each step's D2H copy overlapping the next "
                            "step's traversal (double-buffered outputs)",
                    "serial_value": ser_value, "host_copies_match_device": e2e_ok},
            "clocks": clk.summary(), "gpu_launches": my_launches, "verified": verified,
            "next3_direction_optimising": next3,
        }
        if next4 is not None:
            line["next4_one_traversal_over_ranks"] = next4
        print(json.dumps(line), flush=True)
        if args.detail_out:
            def d8(stt):
                # per level, work vs gap (globaltimer stamps of the captured
                # loop; t_begin = the previous level's end).  Tier 1: gap = until k_explore's
                # CTA 0 starts, work = k_explore + k_compact; tiers 0 / cluster run inside one
                # launch, so their whole span is work (gap 0 except the first level).
                out = []
                for r in stt:
                    t0_, t1_ = int(r["t_begin_ns"]), int(r["t_end_ns"])
                    xb, xe = int(r["t_explore_begin_ns"]), int(r["t_explore_end_ns"])
                    rec = {"l": int(r["level"]), "n_l": int(r["n_l"]), "e_l": int(r["e_l"]),
                           "tier": int(r["tier"]), "grid": int(r["grid"]),
                           "candidates": int(r["candidates"]), "kept": int(r["kept"]),
                           "passes": max(1, int(r["pad"])) if int(r["tier"]) == 1 else 1}
                    if int(r["tier"]) in (1, 3) and xb > 0:
                        rec.update(gap_us=(xb - t0_) / 1e3, work_us=(t1_ - xb) / 1e3,
                                   explore_us=(xe - xb) / 1e3 if xe > xb else None,
                                   compact_us=(t1_ - xe) / 1e3 if xe > xb else None)
                    else:
                        rec.update(gap_us=0.0, work_us=(t1_ - t0_) / 1e3)
                    out.append(rec)
                return out
            detail["per_source"] = {int(s): {"m_c": p["m_c"], "levels": p["levels"],
                                             "launches": p["launches"],
                                             "per_level": d8(p["stats"])}
                                    for s, p in per.items()}
            detail["step_ms"] = step_ms
            detail["per_step_gteps"] = per_step_gteps
            with open(args.detail_out, "w") as f:
                json.dump(detail, f, default=lambda o: o.item() if hasattr(o, "item") else str(o))
    bfs.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())

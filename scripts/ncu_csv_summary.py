"""Summaries of ncu --csv metric logs (runs here, no GPU).
  launches: per-kernel launch count, total and mean device time, share of the total
  traffic:  mean DRAM read+write bytes per k_explore launch (the roofline's `traffic`)"""
import csv
import io
import json
import sys
from collections import defaultdict


def rows(path):
    text = open(path).read()
    start = text.index('"ID"')
    return list(csv.DictReader(io.StringIO(text[start:])))


def scale(v, unit):
    v = float(v.replace(",", ""))
    return v * {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0,
                "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0,
                "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1.0)


STEP_KERNELS = ("k_init", "k_dispatch", "k_small", "k_explore", "k_compact", "k_finalize")


def launches(path):
    """Traversal-step kernels only (create-time preprocessing and torch's own kernels of the
    harness are listed in the raw CSV but are not part of a step)."""
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows(path):
        if r["Metric Name"] == "gpu__time_duration.sum":
            # "void s3bfs::k_explore<0>(s3bfs::Params)" -> "k_explore"
            k = r["Kernel Name"].split("(")[0].split("<")[0].replace("void ", "")
            k = k.replace("s3bfs::", "").strip()
            if k not in STEP_KERNELS:
                continue
            agg[k][0] += 1
            agg[k][1] += scale(r["Metric Value"], r["Metric Unit"])
    tot = sum(v[1] for v in agg.values()) or 1.0
    return {k: {"launches": v[0], "total_ms": v[1] * 1e3, "mean_us": v[1] / v[0] * 1e6,
                "share": v[1] / tot} for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])}


def traffic(path):
    per = defaultdict(dict)
    for r in rows(path):
        per[r["ID"]][r["Metric Name"]] = scale(r["Metric Value"], r["Metric Unit"])
    recs = [v for v in per.values() if "dram__bytes_read.sum" in v]
    b = [v["dram__bytes_read.sum"] + v["dram__bytes_write.sum"] for v in recs]
    t = [v["gpu__time_duration.sum"] for v in recs]
    return {"launches": len(recs), "bytes_per_launch": sum(b) / len(b),
            "mean_ms": sum(t) / len(t) * 1e3, "dram_gbs_under_ncu": sum(b) / sum(t) / 1e9}


if __name__ == "__main__":
    kind, path = sys.argv[1], sys.argv[2]
    print(json.dumps(launches(path) if kind == "launches" else traffic(path), indent=1))

"""Summarise an ncu --csv metric capture of k_explore launches into profiles/ncu_traffic.json
(keyed by config, read by bench.py for roofline.traffic).
usage: python scripts/ncu_traffic.py CONFIG gpurun_out/traffic.csv [--out profiles/ncu_traffic.json]
Metrics expected per launch: dram__bytes_read.sum, dram__bytes_write.sum,
gpu__time_duration.sum, lts__t_sector_hit_rate.pct (l1tex__t_sector_hit_rate.pct optional)."""
import csv
import json
import os
import sys
from collections import defaultdict

cfg, path = sys.argv[1], sys.argv[2]
out = sys.argv[sys.argv.index("--out") + 1] if "--out" in sys.argv else "profiles/ncu_traffic.json"
rows = [l for l in open(path) if l.startswith('"')]
launch = defaultdict(dict)
for r in csv.DictReader(rows):
    if "k_explore" not in r["Kernel Name"]:
        continue
    v = float(r["Metric Value"].replace(",", ""))
    unit = r["Metric Unit"]
    if r["Metric Name"] == "gpu__time_duration.sum":
        v = v * {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3}.get(unit, 1.0)
    elif unit in ("Kbyte", "Mbyte", "Gbyte"):
        v = v * {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[unit]
    launch[r["ID"]][r["Metric Name"]] = v
L = [m for m in launch.values() if "dram__bytes_read.sum" in m]
n = len(L)
rd = sum(m["dram__bytes_read.sum"] for m in L)
wr = sum(m["dram__bytes_write.sum"] for m in L)
ms = sum(m["gpu__time_duration.sum"] for m in L)
wt = [m["gpu__time_duration.sum"] for m in L]
l2 = sum(m.get("lts__t_sector_hit_rate.pct", 0) * w for m, w in zip(L, wt)) / max(ms, 1e-12)
l1 = sum(m.get("l1tex__t_sector_hit_rate.pct", 0) * w for m, w in zip(L, wt)) / max(ms, 1e-12)
peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6549.8
rec = {"kernel": "k_explore", "launches": n, "dram_bytes_per_launch": (rd + wr) / n,
       "dram_read_bytes_per_launch": rd / n, "dram_write_bytes_per_launch": wr / n,
       "mean_ms_under_ncu": ms / n, "dram_gbs_under_ncu": (rd + wr) / (ms / 1e3) / 1e9,
       "dram_frac_of_measured_peak": (rd + wr) / (ms / 1e3) / 1e9 / peak,
       "dram_frac_of_8tbs": (rd + wr) / (ms / 1e3) / 1e9 / 8000.0,
       "l2_hit_pct_time_weighted": l2, "l1_hit_pct_time_weighted": l1,
       "source": os.path.basename(path),
       "note": "ncu per-launch values are cold-cache and serialised; compare shares/bytes, "
               "not absolute times, with the bench line"}
db = json.load(open(out)) if os.path.exists(out) else {}
if "launches" in db and not isinstance(db.get("launches"), dict):  # round-1 flat layout
    db = {"rmat24_r01": db}
db[cfg] = rec
json.dump(db, open(out, "w"), indent=1)
print(json.dumps(rec, indent=1))

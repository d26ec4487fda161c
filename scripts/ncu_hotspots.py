"""Top SASS hotspots (warp-stall samples) of one kernel launch in an ncu report."""
import csv
import io
import subprocess
import sys

rep, kernel = sys.argv[1], sys.argv[2]
skip = int(sys.argv[3]) if len(sys.argv) > 3 else 0
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
out = subprocess.check_output(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                               "sass", "--kernel-name", kernel, "--launch-skip", str(skip),
                               "--launch-count", "1"], text=True, stderr=subprocess.DEVNULL)
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ia, isrc, iss = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
data = [(int(r[iss] or 0), r[ia][-5:], r[isrc].strip()) for r in rows[2:] if len(r) > iss and r[iss].isdigit()]
tot = sum(d[0] for d in data) or 1
order = sorted(range(len(data)), key=lambda i: -data[i][0])[:top]
for i in sorted(order):
    s, a, src = data[i]
    print(f"{100.0 * s / tot:5.1f}%  {a}  {src[:90]}")

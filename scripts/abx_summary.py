"""Summarise scripts/abx.sh logs: per variant the runs' GTEPS, k_explore/k_compact us, frac."""
import collections
import re
import sys

for f in sys.argv[1:]:
    vals = collections.defaultdict(list)
    for line in open(f):
        m = re.match(r"x/(\S+)\s+GTEPS\s+([\d.]+)\s+kx\s+([\d.]+) us kc\s+([\d.]+) us frac\S+ \S+ ([\d.]+)", line)
        if m:
            vals[m.group(1)].append(tuple(float(m.group(i)) for i in range(2, 6)))
    print(f)
    for k, v in vals.items():
        v = sorted(v)
        print(f"  {k:14s}", " | ".join(f"{a:7.2f} kx={b:6.0f} kc={c:5.0f} frac={d:.3f}" for a, b, c, d in v))

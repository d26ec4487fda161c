# Process-level A/B (experiment driver): one library per process, variants alternating over
# ROUNDS rounds, so no variant pays for being the second CUDA module loaded in a process
# (measured: the second of two different libraries loaded in one process runs 2-10 % slower).
# usage: ROUNDS=3 bash scripts/ab.sh CONFIG NSRC tag=lib.so [tag=lib.so ...]
cfg=$1; nsrc=$2; shift 2
out=gpurun_out/ab_${cfg}.log
: > $out
for r in $(seq ${ROUNDS:-3}); do
  for v in "$@"; do
    VARIANT_OPTS=${VARIANT_OPTS:-'{"default": {}}'} ROUNDS=1 timeout 300 python scripts/variants.py $cfg $nsrc $v 2>&1 | grep GTEPS >> $out
  done
done
python - "$out" <<'EOF'
import re, sys, collections
vals = collections.defaultdict(list)
for line in open(sys.argv[1]):
    m = re.match(r"(\S+)\s+GTEPS\s+([\d.]+)", line)
    if m:
        vals[m.group(1)].append(float(m.group(2)))
for k, v in vals.items():
    v = sorted(v)
    print(f"{sys.argv[1].split('ab_')[1][:-4]:8s} {k:28s} median {v[len(v)//2]:8.3f}  runs {' '.join(f'{x:.3f}' for x in v)}")
EOF

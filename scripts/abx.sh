# Process-level A/B over (library, option set) pairs: every pair in its own process, pairs
# alternating over ROUNDS rounds.  usage:
#   ROUNDS=3 bash scripts/abx.sh CONFIG NSRC OUT 'name|lib.so|{"opt": v}' ...
cfg=$1; nsrc=$2; out=$3; shift 3
: > $out
for r in $(seq ${ROUNDS:-3}); do
  for spec in "$@"; do
    name=${spec%%|*}; rest=${spec#*|}; lib=${rest%%|*}; js=${rest#*|}
    VARIANT_OUT=/dev/null VARIANT_OPTS="{\"$name\": $js}" ROUNDS=1 timeout 600 \
      python scripts/variants.py $cfg $nsrc x=$lib 2>&1 | grep -E "GTEPS|src" >> $out
  done
done
python - "$out" <<'PY'
import re, sys, collections
vals, kx = collections.defaultdict(list), collections.defaultdict(list)
for line in open(sys.argv[1]):
    m = re.match(r"x/(\S+)\s+GTEPS\s+([\d.]+)\s+kx\s+([\d.]+)", line)
    if m:
        vals[m.group(1)].append(float(m.group(2))); kx[m.group(1)].append(float(m.group(3)))
for k, v in vals.items():
    i = sorted(range(len(v)), key=lambda j: v[j])[len(v) // 2]
    print(f"{k:24s} GTEPS median {v[i]:8.2f} (kx {kx[k][i]:7.0f} us)  runs {' '.join(f'{x:.2f}' for x in sorted(v))}")
PY

# Process-level A/B over OPTION sets of one library (experiment driver): each option set in its
# own process, alternating over ROUNDS rounds (no handle-order bias inside a process).
# usage: ROUNDS=3 bash scripts/opts_ab.sh CONFIG NSRC LIB 'name={"k": v}' 'name2={...}' ...
cfg=$1; nsrc=$2; lib=$3; shift 3
out=gpurun_out/optab_${cfg}.log
: > $out
for r in $(seq ${ROUNDS:-3}); do
  for o in "$@"; do
    name=${o%%=*}; js=${o#*=}
    VARIANT_OPTS="{\"$name\": $js}" ROUNDS=1 timeout 300 python scripts/variants.py $cfg $nsrc cur=$lib 2>&1 | grep GTEPS >> $out
  done
done
python - "$out" <<'EOF'
import re, sys, collections
vals = collections.defaultdict(list)
for line in open(sys.argv[1]):
    m = re.match(r"\S+/(\S+)\s+GTEPS\s+([\d.]+)", line)
    if m:
        vals[m.group(1)].append(float(m.group(2)))
for k, v in vals.items():
    v = sorted(v)
    print(f"{sys.argv[1].split('optab_')[1][:-4]:8s} {k:20s} median {v[len(v)//2]:8.3f}  runs {' '.join(f'{x:.3f}' for x in v)}")
EOF

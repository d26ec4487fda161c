# bench line per BASELINE config (experiment record, not the driver's bench)
for cfg in ${CFGS:-rmat24 rmat20 er grid tail}; do
  python bench.py --config $cfg --steps ${STEPS:-32} --warmup 3 --oracle-sources ${ORS:-1} --direction ${DIR:-0} --detail-out gpurun_out/detail_${cfg}_d${DIR:-0}.json > gpurun_out/bench_${cfg}_d${DIR:-0}.log 2>&1
  python -c "import json; l=json.loads(open('gpurun_out/bench_${cfg}_d${DIR:-0}.log').read().strip().splitlines()[-1]); print('$cfg', 'dir=${DIR:-0}', round(l['value'],3), 'GTEPS', round(l['ms_per_step'],4), 'ms', 'roof', round(l['roofline']['frac'],3), l['verified'])"
done

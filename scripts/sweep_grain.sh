for cfg in rmat24 rmat20 er tail; do
for g in 16384 8192 4096 2048 1024; do
  python bench.py --config $cfg --steps 32 --warmup 3 --oracle-sources 0 --grain $g > gpurun_out/sweep_${cfg}_${g}.log 2>&1
  python -c "import json,sys; l=json.loads(open('gpurun_out/sweep_${cfg}_${g}.log').read().strip().splitlines()[-1]); print('$cfg', $g, round(l['value'],2), round(l['ms_per_step'],4))"
done; done

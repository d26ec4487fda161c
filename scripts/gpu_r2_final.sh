# round-2 evidence at HEAD: GPU tests, smoke, default bench, all configs, launch list, traffic,
# ncu full capture of k_explore / k_compact (R-MAT 24 source 0, host loop)
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build_rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo bench_rc=$?
tail -1 gpurun_out/bench_default.log | cut -c1-300
: > gpurun_out/bench_all_configs.jsonl
for cfg in er grid rmat20 tail; do
  timeout 600 python bench.py --config $cfg --steps 32 --warmup 3 --oracle-sources 2 --detail-out gpurun_out/d8_$cfg.json > gpurun_out/bench_$cfg.log 2>&1
  tail -1 gpurun_out/bench_$cfg.log >> gpurun_out/bench_all_configs.jsonl
done
tail -1 gpurun_out/bench_default.log >> gpurun_out/bench_all_configs.jsonl
python bench.py --steps 4 --warmup 3 --oracle-sources 0 --no-next3 > gpurun_out/bench_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 4 --warmup 3 --oracle-sources 0 --no-next3 \
    > gpurun_out/ncu_launch.log 2>&1
echo launches_rc=$?
python scripts/prof_run.py --all > gpurun_out/prof_all_plain.log 2>&1 && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,l1tex__t_sector_hit_rate.pct \
    --clock-control none -k regex:k_explore --csv --log-file gpurun_out/traffic.csv \
    python scripts/prof_run.py --all > gpurun_out/ncu_traffic.log 2>&1
echo traffic_rc=$?
python scripts/prof_run.py > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_explore|k_compact" -c 5 \
    -o gpurun_out/r2_prof_final -f python scripts/prof_run.py > gpurun_out/ncu_full.log 2>&1
echo ncu_rc=$?
python scripts/prof_run.py --config grid > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_small|k_cluster" -c 2 \
    -o gpurun_out/r2_prof_grid -f python scripts/prof_run.py --config grid > gpurun_out/ncu_grid.log 2>&1
echo ncu_grid_rc=$?

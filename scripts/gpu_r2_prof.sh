mkdir -p gpurun_out
python scripts/prof_run.py > gpurun_out/r2_prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_explore -c 4 -f -o gpurun_out/r2_prof_kx \
    python scripts/prof_run.py > gpurun_out/r2_ncu_full.log 2>&1
echo full_rc=$?
python bench.py --steps 3 --warmup 3 --no-next3 --oracle-sources 0 > gpurun_out/r2_bench_small.log 2>&1 && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,l1tex__t_sector_hit_rate.pct \
    --clock-control none -k regex:k_explore --csv --log-file gpurun_out/r2_traffic_rmat24.csv \
    python bench.py --steps 3 --warmup 3 --no-next3 --oracle-sources 0 > gpurun_out/r2_ncu_traffic.log 2>&1
echo traffic_rc=$?
tail -c 1500 gpurun_out/r2_bench_small.log

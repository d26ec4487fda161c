# ncu evidence for the bench line: launch list of the bench command + k_explore DRAM traffic
set -x
python bench.py --steps 4 --warmup 3 --oracle-sources 0 > gpurun_out/bench_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 4 --warmup 3 --oracle-sources 0 \
    > gpurun_out/ncu_launch.log 2>&1
echo launches_rc=$?
python scripts/prof_run.py --all > gpurun_out/prof_all_plain.log 2>&1 && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct \
    --clock-control none -k regex:k_explore --csv --log-file gpurun_out/traffic.csv \
    python scripts/prof_run.py --all > gpurun_out/ncu_traffic.log 2>&1
echo traffic_rc=$?

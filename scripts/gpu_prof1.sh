set -x
python scripts/prof_run.py > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_explore -s 1 -c 2 -o gpurun_out/prof_explore -f python scripts/prof_run.py > gpurun_out/ncu_explore.log 2>&1
echo ncu_rc=$?
python bench.py --steps 4 --warmup 3 --oracle-sources 0 > gpurun_out/bench_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 4 --warmup 3 --oracle-sources 0 > gpurun_out/ncu_launch.log 2>&1
echo ncu2_rc=$?
tail -3 gpurun_out/ncu_explore.log

set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo bench_rc=$?
tail -1 gpurun_out/bench_default.log | cut -c1-400
STEPS=32 bash scripts/bench_configs.sh > gpurun_out/cfgs_d0.txt 2>&1
DIR=1 STEPS=32 bash scripts/bench_configs.sh > gpurun_out/cfgs_d1.txt 2>&1
cat gpurun_out/cfgs_d0.txt gpurun_out/cfgs_d1.txt
bash scripts/gpu_evidence.sh > gpurun_out/evidence.log 2>&1; tail -3 gpurun_out/evidence.log
python scripts/prof_run.py > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_explore|k_compact" -c 6 -o gpurun_out/prof_final2 -f python scripts/prof_run.py > gpurun_out/ncu_full.log 2>&1; echo ncu_rc=$?

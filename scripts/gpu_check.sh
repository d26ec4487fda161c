set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc; free -g | head -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
timeout 900 python -m pytest tests -m gpu -x -q -k "not rmat24 and not 2_pow_28" > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
timeout 600 python bench.py --steps 16 --warmup 3 --detail-out gpurun_out/bench_detail.json > gpurun_out/bench.log 2>&1; echo bench_rc=$?
tail -5 gpurun_out/pytest_gpu.log; tail -3 gpurun_out/bench.log

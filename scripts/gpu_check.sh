# one gpurun call: smoke, the GPU test suite, a bench line, then (NCU=1) ncu of k_explore
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
timeout 1200 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
timeout 600 python bench.py --steps ${STEPS:-32} --warmup 5 --detail-out gpurun_out/bench_detail.json > gpurun_out/bench.log 2>&1; echo bench_rc=$?
tail -4 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/bench.log | cut -c1-1500
if [ -n "$NCU" ]; then
python scripts/prof_run.py > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"${NCU_K:-k_explore}" -s ${NCU_S:-1} -c ${NCU_C:-2} -o gpurun_out/prof_${NCU_K:-k_explore} -f python scripts/prof_run.py > gpurun_out/ncu.log 2>&1
echo ncu_rc=$?
fi

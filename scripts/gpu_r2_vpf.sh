# GPU tests at HEAD; k_explore L2 prefetch of discovered records (for k_compact) A/B;
# D8 per-level work/gap detail of the small-level configs
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gpu_tests.log 2>&1; rc=$?; echo "tests rc=$rc"; tail -3 gpurun_out/r2_gpu_tests.log
[ $rc -eq 0 ] || exit 1
L=paper_2209_08764_b200/libs3bfs.so
ROUNDS=3 bash scripts/abx.sh rmat24 8 gpurun_out/r2_vpf_rmat24.log "base|$L|{}" "vpf|variants/libs3bfs_vpf.so|{}"
ROUNDS=2 bash scripts/abx.sh rmat20 8 gpurun_out/r2_vpf_rmat20.log "base|$L|{}" "vpf|variants/libs3bfs_vpf.so|{}"
python scripts/abx_summary.py gpurun_out/r2_vpf_*.log
for cfg in er grid rmat20 tail; do
  python bench.py --config $cfg --steps 16 --warmup 3 --oracle-sources 1 --no-next3 --detail-out gpurun_out/d8_$cfg.json > gpurun_out/bench_$cfg.log 2>&1
  tail -1 gpurun_out/bench_$cfg.log | cut -c1-200
done

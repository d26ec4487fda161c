# k_small on-chip Owner table (one L2 round trip per tier-0 level fewer) vs the L2 Owner check
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gpu_tests.log 2>&1; rc=$?; echo "tests rc=$rc"; tail -3 gpurun_out/r2_gpu_tests.log
[ $rc -eq 0 ] || exit 1
L=paper_2209_08764_b200/libs3bfs.so
ROUNDS=3 bash scripts/abx.sh grid 2 gpurun_out/r2_ks_grid.log "ks0|variants/libs3bfs_ks0.so|{}" "onchip|$L|{}"
ROUNDS=3 bash scripts/abx.sh er 8 gpurun_out/r2_ks_er.log "ks0|variants/libs3bfs_ks0.so|{}" "onchip|$L|{}"
ROUNDS=2 bash scripts/abx.sh tail 4 gpurun_out/r2_ks_tail.log "ks0|variants/libs3bfs_ks0.so|{}" "onchip|$L|{}"
ROUNDS=2 bash scripts/abx.sh rmat20 8 gpurun_out/r2_ks_rmat20.log "ks0|variants/libs3bfs_ks0.so|{}" "onchip|$L|{}"
ROUNDS=2 bash scripts/abx.sh rmat24 4 gpurun_out/r2_ks_rmat24.log "ks0|variants/libs3bfs_ks0.so|{}" "onchip|$L|{}"
python scripts/abx_summary.py gpurun_out/r2_ks_*.log

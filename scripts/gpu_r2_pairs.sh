mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gpu_tests.log 2>&1; rc=$?; echo "tests rc=$rc"; tail -5 gpurun_out/r2_gpu_tests.log
[ $rc -eq 0 ] || exit 1
L=paper_2209_08764_b200/libs3bfs.so
ROUNDS=2 bash scripts/abx.sh rmat24 8 gpurun_out/r2_pairs_rmat24.log "r01|variants/libs3bfs_r01.so|{}" "modes|variants/libs3bfs_modes.so|{\"hub_vertices\": 524288}" "pairs0|variants/libs3bfs_pairs0.so|{}" "pairs|$L|{}" "pairs-never|$L|{\"tag_mode_pct\": -1}"
ROUNDS=1 bash scripts/abx.sh rmat20 8 gpurun_out/r2_pairs_rmat20.log "r01|variants/libs3bfs_r01.so|{}" "pairs0|variants/libs3bfs_pairs0.so|{}" "pairs|$L|{}" "pairs-never|$L|{\"tag_mode_pct\": -1}"
ROUNDS=1 bash scripts/abx.sh er 8 gpurun_out/r2_pairs_er.log "r01|variants/libs3bfs_r01.so|{}" "pairs|$L|{}" "pairs-never|$L|{\"tag_mode_pct\": -1}"
python scripts/abx_summary.py gpurun_out/r2_pairs_*.log
grep src gpurun_out/r2_pairs_rmat24.log | head -12

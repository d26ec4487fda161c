mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/r2_gpu_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r2_gpu_tests.log
L=paper_2209_08764_b200/libs3bfs.so
R=variants/libs3bfs_r01.so
ROUNDS=3 bash scripts/abx.sh rmat24 8 gpurun_out/r2_modes_rmat24.log "r01|$R|{}" "new-default|$L|{}" "new-never|$L|{\"tag_mode_pct\": -1}" "new-always|$L|{\"tag_mode_pct\": 101}" "new-hub19|$L|{\"hub_vertices\": 524288}" "new-pct60|$L|{\"tag_mode_pct\": 60}"
ROUNDS=2 bash scripts/abx.sh rmat20 8 gpurun_out/r2_modes_rmat20.log "r01|$R|{}" "new-default|$L|{}" "new-never|$L|{\"tag_mode_pct\": -1}" "new-always|$L|{\"tag_mode_pct\": 101}"

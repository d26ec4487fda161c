mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/r2_gpu_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r2_gpu_tests.log
L=paper_2209_08764_b200/libs3bfs.so
R=variants/libs3bfs_r01.so
ROUNDS=2 bash scripts/abx.sh rmat24 8 gpurun_out/r2_modes2_rmat24.log "r01|$R|{}" "new-default|$L|{}" "new-pct90|$L|{\"tag_mode_pct\": 90}" "new-pct60|$L|{\"tag_mode_pct\": 60}" "new-hub20|$L|{\"hub_vertices\": 1048576}"
ROUNDS=2 bash scripts/abx.sh rmat20 8 gpurun_out/r2_modes2_rmat20.log "r01|$R|{}" "new-default|$L|{}" "new-pct90|$L|{\"tag_mode_pct\": 90}" "new-pct60|$L|{\"tag_mode_pct\": 60}"
ROUNDS=2 bash scripts/abx.sh er 8 gpurun_out/r2_modes2_er.log "r01|$R|{}" "new-default|$L|{}" "new-pct90|$L|{\"tag_mode_pct\": 90}" "new-pct60|$L|{\"tag_mode_pct\": 60}"
ROUNDS=2 bash scripts/abx.sh tail 4 gpurun_out/r2_modes2_tail.log "r01|$R|{}" "new-default|$L|{}"

# programmatic dependent launch between the captured loop's chained kernels vs plain edges
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gpu_tests.log 2>&1; rc=$?; echo "tests rc=$rc"; tail -3 gpurun_out/r2_gpu_tests.log
[ $rc -eq 0 ] || exit 1
L=paper_2209_08764_b200/libs3bfs.so
ROUNDS=3 bash scripts/abx.sh er 8 gpurun_out/r2_pdl_er.log "pdl0|variants/libs3bfs_pdl0.so|{}" "pdl|$L|{}"
ROUNDS=2 bash scripts/abx.sh rmat20 8 gpurun_out/r2_pdl_rmat20.log "pdl0|variants/libs3bfs_pdl0.so|{}" "pdl|$L|{}"
ROUNDS=2 bash scripts/abx.sh grid 2 gpurun_out/r2_pdl_grid.log "pdl0|variants/libs3bfs_pdl0.so|{}" "pdl|$L|{}"
ROUNDS=2 bash scripts/abx.sh tail 4 gpurun_out/r2_pdl_tail.log "pdl0|variants/libs3bfs_pdl0.so|{}" "pdl|$L|{}"
ROUNDS=3 bash scripts/abx.sh rmat24 8 gpurun_out/r2_pdl_rmat24.log "pdl0|variants/libs3bfs_pdl0.so|{}" "pdl|$L|{}"
python scripts/abx_summary.py gpurun_out/r2_pdl_*.log

mkdir -p gpurun_out
python scripts/dbg_small.py variants/libs3bfs_check.so; timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gpu_tests.log 2>&1; rc=$?; echo "tests rc=$rc"; tail -5 gpurun_out/r2_gpu_tests.log
[ $rc -eq 0 ] || exit 1
L=paper_2209_08764_b200/libs3bfs.so
R=variants/libs3bfs_r01.so
ROUNDS=2 bash scripts/abx.sh rmat24 8 gpurun_out/r2_chunk_rmat24.log "r01|$R|{}" "chunk|$L|{}" "chunk-never|$L|{\"tag_mode_pct\": -1}" "chunk-pct60|$L|{\"tag_mode_pct\": 60}"
ROUNDS=2 bash scripts/abx.sh rmat20 8 gpurun_out/r2_chunk_rmat20.log "r01|$R|{}" "chunk|$L|{}" "chunk-never|$L|{\"tag_mode_pct\": -1}"
ROUNDS=2 bash scripts/abx.sh er 8 gpurun_out/r2_chunk_er.log "r01|$R|{}" "chunk|$L|{}" "chunk-never|$L|{\"tag_mode_pct\": -1}"
ROUNDS=1 bash scripts/abx.sh tail 4 gpurun_out/r2_chunk_tail.log "r01|$R|{}" "chunk|$L|{}"
python scripts/abx_summary.py gpurun_out/r2_chunk_*.log
